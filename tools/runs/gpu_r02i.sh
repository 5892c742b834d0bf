#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02i}
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > $O/${T}_sharded_tests.log 2>&1; echo "rc=$?" >> $O/${T}_sharded_tests.log
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "test_gpu_matches_reference_golden and (p2_sift or p4_gist or p2_wide) and file and (auto or generic)" > $O/${T}_san_${tool}.log 2>&1; echo "rc=$?" >> $O/${T}_san_${tool}.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_sharded.py -x -q -k "p2_small and 3" > $O/${T}_san_memcheck_sharded.log 2>&1; echo "rc=$?" >> $O/${T}_san_memcheck_sharded.log
echo done
