# sharded protocol: tests + the SIFT1B 8-rank simulation bench line
O=gpurun_out; T=${1:-sq}
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_topk.py -x -q > $O/${T}_tests.log 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sim8.json 2> $O/${T}_sim8.err
