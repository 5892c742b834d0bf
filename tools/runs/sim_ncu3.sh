O=gpurun_out; T=${1:-sn}
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:"rerank_ij" -c 1 -f -o $O/${T}_small \
  python bench.py --workload sift1b --sim-ranks 8 --steps 1 --warmup 3 --no-recall --no-cpu-baseline > $O/${T}_sim.log 2>&1
