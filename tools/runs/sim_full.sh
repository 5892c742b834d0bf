# full GPU suite + the SIFT1B 8-rank simulation bench line
O=gpurun_out; T=${1:-sf}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sim8.json 2> $O/${T}_sim8.err
