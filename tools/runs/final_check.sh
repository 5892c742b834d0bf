# the committed state: full GPU suite + smoke + one default bench line
O=gpurun_out; T=${1:-fc}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err
