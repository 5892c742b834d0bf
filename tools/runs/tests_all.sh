O=gpurun_out; T=${1:-ta}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sim8.json 2> $O/${T}_sim8.err
timeout 300 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat.json 2>$O/${T}_lat.err
