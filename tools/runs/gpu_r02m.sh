#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02m}
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_topk.py -x -q -k "sift1b or sharded" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall --no-cpu-baseline --variant 2 > $O/${T}_sift1b_v2.json 2> $O/${T}_sift1b_v2.err
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
echo done
