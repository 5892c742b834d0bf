# per-kernel times of the SIFT1B 8-rank protocol (rank 0, peers simulated): ncu launch list of the
# query kernels only (cold-cache, serialised)
O=gpurun_out; T=${1:-sn}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled \
  -k regex:"rerank|fine_lut|move_ranges|scan_counts|copy_segments|merge_ranked|traverse_warp_wide|binsel_par" -c 60 \
  --csv --log-file $O/${T}_sim_launches.csv \
  python bench.py --workload sift1b --sim-ranks 8 --steps 2 --warmup 3 --no-recall --no-cpu-baseline > $O/${T}_sim.log 2>&1
