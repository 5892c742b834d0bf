# grouped ranking in the split slices: full GPU suite, smoke, latency sweep
O=gpurun_out; T=${1:-fc4}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 900 python tools/latency_sweep.py > $O/${T}_latency_sweep.json 2> $O/${T}_latency_sweep.err
