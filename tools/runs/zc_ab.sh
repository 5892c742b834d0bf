# end-to-end with the queries and results crossing the link inside the kernels (zero-copy) vs copies
O=gpurun_out; T=${1:-zc}
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_dropin_cxx.py -x -q > $O/${T}_tests.log 2>&1
for z in 1 0; do
  for w in deep100m gist1m sift1m; do
    PQTG_ZERO_COPY=$z timeout 900 python bench.py --workload $w --index gpu --steps 20 --warmup 5 --no-cpu-baseline --no-recall > $O/${T}_${w}_z$z.json 2>$O/${T}_${w}_z$z.err
  done
done
