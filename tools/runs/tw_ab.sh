O=gpurun_out; T=${1:-ta}
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > $O/${T}_tests.log 2>&1
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall --no-cpu-baseline > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
timeout 900 python bench.py --workload sift1m --index gpu --steps 20 --warmup 5 --no-recall --no-cpu-baseline > $O/${T}_sift1m.json 2> $O/${T}_sift1m.err
