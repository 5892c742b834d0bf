O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/r02b_gpu_tests.log 2>&1; echo "rc=$?" >> $O/r02b_gpu_tests.log
for w in deep100m sift1m gist1m; do timeout 600 python tools/bank_probe.py $w 100 > $O/r02b_bank_$w.json 2> $O/r02b_bank_$w.err; done
echo done
