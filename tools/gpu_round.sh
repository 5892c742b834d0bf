#!/bin/bash
# One GPU session: parity tests, smoke, bench (both arms), ncu launch list, ncu --set full capture.
# usage: tools/gpu_round.sh TAG [extra bench args]
TAG=${1:-r01}; shift
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py "$@" > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:pqtg \
  --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-recall "$@" > $O/${TAG}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"traverse|binsel|rerank" -c 6 -f -o $O/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall "$@" > $O/${TAG}_ncu_full.log 2>&1
echo done
