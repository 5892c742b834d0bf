#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02n}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
for plan in "" "1,1,1,1,1,1,1,1" "1,1"; do
  PQTG_CHUNK_PLAN=$plan timeout 600 python bench.py --workload deep100m --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_deep_plan${plan//,/}.json 2> $O/${T}_deep_plan${plan//,/}.err
done
echo done
