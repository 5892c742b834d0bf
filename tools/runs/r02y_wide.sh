#!/bin/bash
# 256-bit code-row loads in the re-rank: parity suites, then A/B against 16-byte loads
O=gpurun_out; mkdir -p $O; T=${1:-wd1}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_sharded.py tests/test_gpu_topk.py -x -q > $O/${T}_parity.log 2>&1; echo "rc=$?" >> $O/${T}_parity.log
for w in sift1m deep100m; do
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_wide.json 2> $O/${T}_${w}_wide.err
  PQTG_RERANK=narrow timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_narrow.json 2> $O/${T}_${w}_narrow.err
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_wide2.json 2> $O/${T}_${w}_wide2.err
done
M=l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:rerank -c 1 --csv python bench.py --workload sift1m --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu_sift1m_wide.csv 2> $O/${T}_ncu_sift1m_wide.err
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
echo done
