# latency sweep with SM clocks sampled during the device loop + API / drop-in tests
O=gpurun_out; T=${1:-lq}
timeout 300 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat.json 2>$O/${T}_err.txt
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_dropin_cxx.py tests/test_gpu_parity.py -x -q > $O/${T}_tests.log 2>&1
PQTG_PHASES=1 timeout 300 python tools/phase_probe.py sift1m 1 >> $O/${T}_phase.txt 2>>$O/${T}_err.txt
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_edges.py -x -q > $O/${T}_tests2.log 2>&1
