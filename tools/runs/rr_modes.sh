# re-rank table-layout A/B: default (E, c2) float2 table vs split 4-byte tables (PQTG_RERANK=split)
O=gpurun_out; T=${1:-rm}
PQTG_RERANK=split timeout 900 python -m pytest tests -x -q -m gpu -k "parity or topk or edges" > $O/${T}_tests_split.log 2>&1
for m in default split; do
  for w in sift1m deep100m; do
    PQTG_RERANK=$m timeout 900 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_${m}.json 2>$O/${T}_${w}_${m}.err
  done
done
PQTG_RERANK=split timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -k regex:rerank -c 1 -f -o $O/${T}_split_full python bench.py --workload deep100m --index gpu --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu.log 2>&1
