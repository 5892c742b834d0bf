#!/bin/bash
# SIFT1B shard 0 of 8 with the oracle shard-view parity; the sharded bench path on one rank
O=gpurun_out; mkdir -p $O; T=${1:-r02e}
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
timeout 600 python bench.py --workload sift1m --index gpu --shard --steps 10 --warmup 3 --no-recall > $O/${T}_sift1m_shard1.json 2> $O/${T}_sift1m_shard1.err
echo done
