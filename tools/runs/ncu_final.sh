# ncu --set full of the committed re-rank on DEEP100M (one launch per stage, --chunks 1)
O=gpurun_out; T=${1:-nf}
timeout 1500 python bench.py --impl reference --workload deep100m --build-index-only > $O/${T}_build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"traverse|binsel|rerank" -c 3 -f -o $O/${T}_deep_full python bench.py --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu_full.log 2>&1
echo done
