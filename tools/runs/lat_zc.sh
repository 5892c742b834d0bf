O=gpurun_out; T=${1:-lz}
for m in 64 256 1024; do
  PQTG_ZC_MAX=$m timeout 300 python tools/latency_sweep.py --sizes 1,10,100,200,1000 --no-cpu > $O/${T}_zc$m.json 2>>$O/${T}_err.txt
done
