#!/bin/bash
# Quick GPU iteration: parity tests, bench (no CPU leg), ncu --set full of the three query kernels.
# usage: tools/gpu_quick.sh TAG [extra bench args]
TAG=${1:-q}; shift
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${TAG}_gpu_tests.log
tail -3 $O/${TAG}_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline "$@" > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
cat $O/${TAG}_bench.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"traverse|binsel|rerank|screen" -c 4 -f -o $O/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall --chunks 1 "$@" > $O/${TAG}_ncu_full.log 2>&1
echo done
