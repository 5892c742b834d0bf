# re-rank phase clocks + per-query in-kernel stage times at small batches (tools/phase_probe.py)
O=gpurun_out; T=${1:-pp}
for b in 1 100; do
  PQTG_PHASES=1 timeout 300 python tools/phase_probe.py sift1m $b >> $O/${T}_default.txt 2>>$O/${T}_err.txt
  PQTG_PHASES=1 PQTG_SPLIT=1 timeout 300 python tools/phase_probe.py sift1m $b >> $O/${T}_split.txt 2>>$O/${T}_err.txt
done
