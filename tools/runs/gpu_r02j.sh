#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02j}
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "test_gpu_matches_reference_golden and (p2_sift or p4_gist or p2_wide) and file and (auto or generic)" > $O/${T}_san_racecheck.log 2>&1; echo "rc=$?" >> $O/${T}_san_racecheck.log
for w in deep100m sift1m gist1m; do
  for m in default c3; do
    PQTG_RERANK=$m timeout 600 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_${m}.json 2> $O/${T}_${w}_${m}.err
  done
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pqtg|copy|fine|scan|move" --csv --log-file $O/${T}_sim_launches.csv python bench.py --workload sift1b --sim-ranks 8 --steps 3 --warmup 3 --no-recall > $O/${T}_sim_ncu.log 2>&1
echo done
