#!/bin/bash
# re-rank ILP variants: parity under each, then A/B against the default in one run
O=gpurun_out; mkdir -p $O; T=${1:-il1}
for m in half onecta; do
  PQTG_RERANK=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > $O/${T}_parity_$m.log 2>&1; echo "rc=$?" >> $O/${T}_parity_$m.log
done
for w in sift1m deep100m; do
  for m in base half onecta base2; do
    e=$m; [ $m = base ] || [ $m = base2 ] && e=""
    PQTG_RERANK=$e timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_$m.json 2> $O/${T}_${w}_$m.err
  done
done
echo done
