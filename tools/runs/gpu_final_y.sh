#!/bin/bash
# Round-2 final measurement set, in the driver's order: GPU tests, smoke, the reference arm (it
# builds and writes the DEEP100M index), our arm, the ncu launch list and one --set full capture
# (DEEP100M), the other configs, the SIFT1B shard and its 8-rank simulation, the latency sweep,
# (compute-sanitizer is closed on the pool since r02v; its r02v logs stand).  usage: tools/runs/gpu_final.sh TAG
O=gpurun_out; mkdir -p $O; T=${1:-r02y}
{ nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > $O/${T}_box.txt 2>&1
SECONDS=0
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_gpu_tests.log 2>&1; echo "rc=$? ${SECONDS}s" >> $O/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
SECONDS=0
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref.json 2> $O/${T}_ref.err; echo "ref ${SECONDS}s" >> $O/${T}_box.txt; SECONDS=0
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "ours ${SECONDS}s" >> $O/${T}_box.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:pqtg \
  --csv --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-recall > $O/${T}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"traverse|binsel|rerank" -c 3 -f -o $O/${T}_deep_full python bench.py --steps 1 --warmup 3 --chunks 1 --no-cpu-baseline --no-recall > $O/${T}_ncu_full.log 2>&1
for w in sift1m gist1m; do
  timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 > $O/${T}_$w.json 2> $O/${T}_$w.err
done
timeout 1500 python bench.py --workload sift1b --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b.json 2> $O/${T}_sift1b.err
timeout 1500 python bench.py --workload sift1b --sim-ranks 8 --steps 20 --warmup 5 --no-recall > $O/${T}_sift1b_sim8.json 2> $O/${T}_sift1b_sim8.err
timeout 900 python tools/latency_sweep.py > $O/${T}_latency_sweep.json 2> $O/${T}_latency_sweep.err

echo done2
