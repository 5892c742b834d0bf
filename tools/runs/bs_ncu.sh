# ncu --set full (with source) of the SIFT1B tree traversal (W = 128) on the shard-0 workload
O=gpurun_out; T=${1:-tw}
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:"binsel_par" -c 1 -f -o $O/${T}_bs \
  python bench.py --workload sift1b --steps 1 --warmup 3 --chunks 1 --no-recall --no-cpu-baseline > $O/${T}.log 2>&1
