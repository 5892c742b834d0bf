O=gpurun_out; T=${1:-le}
timeout 300 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat.json 2>$O/${T}_err.txt
timeout 600 python -m pytest tests/test_gpu_api.py -x -q > $O/${T}_tests.log 2>&1
timeout 300 python tools/latency_sweep.py --sizes 1,10,100 --no-cpu > $O/${T}_lat2.json 2>>$O/${T}_err.txt
