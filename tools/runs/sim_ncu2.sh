O=gpurun_out; T=${1:-sn}
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none --kernel-name-base mangled \
  -k regex:"fine_lut|scan_counts|move_ranges|copy_segments|merge_ranked" -c 24 \
  --csv --log-file $O/${T}_sim_launches.csv \
  python bench.py --workload sift1b --sim-ranks 8 --steps 2 --warmup 3 --no-recall --no-cpu-baseline > $O/${T}_sim.log 2>&1
