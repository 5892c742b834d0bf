# host-call chunk plans for a 1000-query GIST1M batch (bench e2e line, GPU-built index)
O=gpurun_out; T=${1:-gp}
for plan in "1,1" "1,3" "1,2,1" "1,3,1" "1,4,3" "2,3"; do
  PQTG_CHUNK_PLAN=$plan timeout 600 python bench.py --workload gist1m --index gpu --steps 40 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_$plan.json 2>$O/${T}_$plan.err
done
