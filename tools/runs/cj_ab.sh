O=gpurun_out; T=${1:-cj}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sim8.json 2> $O/${T}_sim8.err
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
