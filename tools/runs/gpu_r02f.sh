#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02f}
timeout 900 python -m pytest tests/test_dropin_cxx.py tests/test_gpu_sharded.py -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 900 python tools/latency_sweep.py --sizes 1,10,100,1000,10000 > $O/${T}_latency.json 2> $O/${T}_latency.err
echo done
