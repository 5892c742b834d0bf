#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02k}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 600 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat.json 2> $O/${T}_lat.err
PQTG_SPLIT=1 timeout 600 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat_split.json 2>&1
PQTG_NO_TRAVERSE_SMALL=1 timeout 600 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat_nosmall.json 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
echo done
