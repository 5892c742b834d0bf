#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02p}
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"traverse|binsel|rerank" -c 3 -f -o $O/${T}_sift1b python bench.py --workload sift1b --steps 1 --warmup 3 --no-cpu-baseline --no-recall --chunks 1 > $O/${T}_ncu.log 2>&1
echo done
