#!/bin/bash
# resort at large budgets (tests + memcheck) and the cooperative row-load re-rank A/B
O=gpurun_out; mkdir -p $O; T=${1:-cp1}
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "resort_large_budget or large_budget" > $O/${T}_resort_tests.log 2>&1; echo "rc=$?" >> $O/${T}_resort_tests.log
PQTG_RERANK=coop timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > $O/${T}_coop_parity.log 2>&1; echo "rc=$?" >> $O/${T}_coop_parity.log
for w in sift1m deep100m; do
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_base.json 2> $O/${T}_${w}_base.err
  PQTG_RERANK=coop timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_coop.json 2> $O/${T}_${w}_coop.err
done
M=l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
for m in base coop; do
  e=""; [ $m = coop ] && e=coop
  PQTG_RERANK=$e timeout 600 ncu --metrics $M --clock-control none -k regex:rerank -c 2 --csv python bench.py --workload sift1m --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu_sift1m_$m.csv 2> $O/${T}_ncu_sift1m_$m.err
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_edges.py -x -q -k "resort_large_budget and 8192 and 2" > $O/${T}_san_memcheck_resort.log 2>&1; echo "rc=$?" >> $O/${T}_san_memcheck_resort.log
echo done
