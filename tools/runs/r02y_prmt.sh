#!/bin/bash
# λ without I2F: parity suites, then A/B against the I2F loop (both with 256-bit row loads)
O=gpurun_out; mkdir -p $O; T=${1:-pm1}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_sharded.py tests/test_gpu_topk.py tests/test_gpu_edges.py -x -q > $O/${T}_parity.log 2>&1; echo "rc=$?" >> $O/${T}_parity.log
for w in deep100m sift1m; do
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_prmt.json 2> $O/${T}_${w}_prmt.err
  PQTG_RERANK=i2f timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_i2f.json 2> $O/${T}_${w}_i2f.err
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_prmt2.json 2> $O/${T}_${w}_prmt2.err
done
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
echo done
