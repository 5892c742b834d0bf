#!/bin/bash
# packed vs scalar re-rank A/B on three workloads (GPU-built indexes), GPU tests, one ncu capture
O=gpurun_out; mkdir -p $O; T=${1:-r02c}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
for w in deep100m sift1m gist1m; do
  for m in scalar packed; do
    PQTG_RERANK=$m timeout 600 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_${m}.json 2> $O/${T}_${w}_${m}.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"rerank" -c 2 -f -o $O/${T}_deep_packed python bench.py --workload deep100m --index gpu --steps 1 --warmup 3 --no-cpu-baseline --no-recall > $O/${T}_ncu.log 2>&1
echo done
