O=gpurun_out; T=${1:-ln}
PQTG_NO_GRAPH=1 timeout 300 python tools/latency_sweep.py --sizes 1,10 --no-cpu > $O/${T}_nograph.json 2>$O/${T}_err.txt
timeout 300 python tools/latency_sweep.py --sizes 1,10 --no-cpu > $O/${T}_graph.json 2>>$O/${T}_err.txt
