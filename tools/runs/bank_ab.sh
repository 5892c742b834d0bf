# per-part bank map of the 1-byte line codes: parity + A/B against the fixed slots
O=gpurun_out; T=${1:-bk}
timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or topk or edges or api or dropin" > $O/${T}_tests.log 2>&1
for m in 1 0; do
  for w in sift1m deep100m; do
    PQTG_BANK_MAP=$m timeout 900 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_map$m.json 2>$O/${T}_${w}_map$m.err
  done
done
timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -k regex:rerank -c 1 -f -o $O/${T}_deep python bench.py --workload deep100m --index gpu --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu.log 2>&1
