#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02r}
for plan in "" "1,2,2,2,2,1" "1,3,3,3,1" "1,2,2,1" "1,4,4,1"; do
  PQTG_CHUNK_PLAN=$plan timeout 600 python bench.py --workload deep100m --index gpu --steps 30 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_deep_plan${plan//,/}.json 2> $O/${T}_deep_plan${plan//,/}.err
done
echo done
