#!/bin/bash
# host-call chunk plans after the faster re-rank (e2e of pqtg_search on pinned buffers)
O=gpurun_out; mkdir -p $O; T=${1:-cp}
for w in deep100m sift1m; do
  for plan in default 1,8,1 1,2,4,2,1 1,6,6,1 2,8,8,2 1,3,3,3,1; do
    if [ $plan = default ]; then pre="env -u PQTG_CHUNK_PLAN"; else pre="env PQTG_CHUNK_PLAN=$plan"; fi
    $pre timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_$plan.json 2> $O/${T}_${w}_$plan.err
  done
done
echo done
