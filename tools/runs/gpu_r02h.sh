#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02h}
PQTG_SPLIT=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"traverse|binsel|rerank" -s 9 -c 3 -f -o $O/${T}_lat1 python tools/latency_sweep.py --sizes 1 --no-cpu > $O/${T}_ncu.log 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
echo done
