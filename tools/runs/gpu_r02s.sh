#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02s}
for c in 1 2 3 4; do
  timeout 600 python bench.py --workload deep100m --index gpu --steps 30 --warmup 5 --no-cpu-baseline --no-recall --chunks $c > $O/${T}_deep_c$c.json 2> $O/${T}_deep_c$c.err
done
timeout 600 python bench.py --workload sift1m --index gpu --steps 30 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_sift1m.json 2> $O/${T}_sift1m.err
echo done
