# latency sweep with SM clocks sampled during the device loop + API / drop-in tests
O=gpurun_out; T=${1:-lq}
timeout 300 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat.json 2>$O/${T}_err.txt
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_dropin_cxx.py tests/test_gpu_parity.py -x -q > $O/${T}_tests.log 2>&1
