O=gpurun_out; T=${1:-ls}
for m in 16 8 12 4; do
  PQTG_SPLIT_MAX=$m timeout 300 python tools/latency_sweep.py --sizes 1,10,50 --no-cpu > $O/${T}_s$m.json 2>>$O/${T}_err.txt
done
