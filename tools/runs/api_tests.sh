O=gpurun_out; T=${1:-at}
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_dropin_cxx.py tests/test_gpu_parity.py -x -q > $O/${T}_tests.log 2>&1
