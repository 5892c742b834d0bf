#!/bin/bash
# DEEP100M (BASELINE configs[2], the N=1 default) as the driver runs it: the reference arm first
# (it builds the index with pqtref on the host CPUs and writes the PQTINDEX file), then our arm
# (reads that file through pqtg_index_load), then the ncu launch list and one --set full capture.
# usage: tools/gpu_deep.sh TAG [extra bench args]
TAG=${1:-r02}; shift
O=gpurun_out
mkdir -p $O
{ nproc; free -g; lscpu | head -20; df -h /tmp; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > $O/${TAG}_box.txt 2>&1
SECONDS=0
timeout 1700 python bench.py --impl reference --steps 5 --warmup 3 "$@" > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
echo "ref arm ${SECONDS}s" >> $O/${TAG}_box.txt; SECONDS=0
timeout 1500 python bench.py --steps 20 --warmup 5 "$@" > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "our arm ${SECONDS}s" >> $O/${TAG}_box.txt; SECONDS=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:pqtg \
  --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-recall "$@" > $O/${TAG}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"traverse|binsel|rerank" -c 6 -f -o $O/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall "$@" > $O/${TAG}_ncu_full.log 2>&1
echo "ncu ${SECONDS}s" >> $O/${TAG}_box.txt
echo done
