#!/bin/bash
O=gpurun_out; mkdir -p $O; T=${1:-r02l}
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_edges.py tests/test_dropin_cxx.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
echo done
