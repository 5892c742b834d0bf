#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02o}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"traverse|binsel|rerank" -s 9 -c 3 -f -o $O/${T}_lat1 python tools/latency_sweep.py --sizes 1 --no-cpu > $O/${T}_ncu.log 2>&1
PQTG_SPLIT=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"traverse|binsel|rerank" -s 9 -c 3 -f -o $O/${T}_lat1_split python tools/latency_sweep.py --sizes 1 --no-cpu > $O/${T}_ncu_split.log 2>&1
timeout 600 nsys --version > /dev/null 2>&1 || true
echo done
