# ncu --set full of the batch-1 re-rank (split slices + merge) on SIFT1M
O=gpurun_out; T=${1:-b1}
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:"rerank_ij" -s 20 -c 1 -f -o $O/${T}_rerank \
  python tools/latency_sweep.py --sizes 1 --no-cpu > $O/${T}.log 2>&1
