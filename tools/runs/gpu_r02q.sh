#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02q}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 600 python bench.py --workload deep100m --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_deep.json 2> $O/${T}_deep.err
echo done
