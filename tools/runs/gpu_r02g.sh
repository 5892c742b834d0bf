#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02g}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 600 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat_split.json 2> $O/${T}_lat_split.err
PQTG_SPLIT=0 timeout 600 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat_nosplit.json 2>&1
PQTG_NO_TRAVERSE_WARP=1 timeout 600 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat_tpart.json 2>&1
echo done
