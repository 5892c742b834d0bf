# re-rank throughput check (GPU-built DEEP100M and SIFT1M)
O=gpurun_out; T=${1:-ab}
for w in sift1m deep100m; do
  timeout 900 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}.json 2>$O/${T}_${w}.err
done
timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -k regex:rerank -c 1 -f -o $O/${T}_deep python bench.py --workload deep100m --index gpu --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu.log 2>&1
