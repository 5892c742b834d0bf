#!/bin/bash
# The other BASELINE.json configs on one GPU: SIFT1M, DEEP100M, GIST1M --exact, SIFT1B shard 0/8,
# and the latency sweep. usage: tools/gpu_workloads.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --workload sift1m > $O/${TAG}_sift1m.json 2> $O/${TAG}_sift1m.err
timeout 900 python bench.py --exact > $O/${TAG}_gist_exact.json 2> $O/${TAG}_gist_exact.err
timeout 1500 python bench.py --workload deep100m --steps 50 > $O/${TAG}_deep100m.json 2> $O/${TAG}_deep100m.err
timeout 1500 python bench.py --workload sift1b --steps 50 --warmup 5 > $O/${TAG}_sift1b.json 2> $O/${TAG}_sift1b.err
timeout 900 python tools/latency_sweep.py > $O/${TAG}_latency_sweep.json 2> $O/${TAG}_latency_sweep.err
echo done
