# small-batch latency: PDL chain, device graph replay, zero-copy results, split re-rank; phase clocks
O=gpurun_out; T=${1:-lp}
timeout 300 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat.json 2>$O/${T}_err.txt
PQTG_SPLIT=0 timeout 300 python tools/latency_sweep.py --sizes 1,10,100,1000 --no-cpu > $O/${T}_lat_split.json 2>>$O/${T}_err.txt
PQTG_CHAIN=0 timeout 300 python tools/latency_sweep.py --sizes 1,10 --no-cpu > $O/${T}_lat_nochain.json 2>>$O/${T}_err.txt
PQTG_CHAIN=all timeout 300 python tools/latency_sweep.py --sizes 1000,10000 --no-cpu > $O/${T}_lat_chainall.json 2>>$O/${T}_err.txt
PQTG_PHASES=1 PQTG_CHAIN=0 timeout 300 python tools/phase_probe.py sift1m 1 >> $O/${T}_phase.txt 2>>$O/${T}_err.txt
PQTG_PHASES=1 timeout 300 python tools/phase_probe.py sift1m 1 >> $O/${T}_phase.txt 2>>$O/${T}_err.txt
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_topk.py -x -q > $O/${T}_tests.log 2>&1
