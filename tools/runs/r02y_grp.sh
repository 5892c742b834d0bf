#!/bin/bash
# top-k ranked within radix bins: parity, then A/B (the grouped DEEP100M run keeps its parity check)
O=gpurun_out; mkdir -p $O; T=${1:-gp1}
PQTG_RERANK=grouped timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_edges.py -x -q > $O/${T}_parity.log 2>&1; echo "rc=$?" >> $O/${T}_parity.log
for w in deep100m sift1m; do
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_base.json 2> $O/${T}_${w}_base.err
  PQTG_RERANK=grouped timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-recall > $O/${T}_${w}_grouped.json 2> $O/${T}_${w}_grouped.err
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_base2.json 2> $O/${T}_${w}_base2.err
done
echo done
