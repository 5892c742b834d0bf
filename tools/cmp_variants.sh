#!/bin/bash
# Parity subset + GIST1M/SIFT1M (and SIFT1B with SIFT1B=1) bench lines per kernel variant.
# usage: VARS="0 3 4" SIFT1B=1 bash tools/cmp_variants.sh
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu -k "parity or topk" 2>&1 | tail -2
for v in ${VARS:-0}; do
python bench.py --no-cpu-baseline --no-recall --variant $v > gpurun_out/gist_v$v.json 2>/dev/null
python bench.py --workload sift1m --no-cpu-baseline --no-recall --variant $v > gpurun_out/sift1m_v$v.json 2>/dev/null
[ -n "$SIFT1B" ] && timeout 900 python bench.py --workload sift1b --steps 50 --warmup 5 --variant $v > gpurun_out/sift1b_v$v.json 2>/dev/null
done
python - <<'PY'
import json
for w in ["gist","sift1m","sift1b"]:
  for v in [0,1,2,3]:
    try:
      d=json.load(open(f"gpurun_out/{w}_v{v}.json")); r=d["roofline"]
      print(w, v, round(d["value"]), round(d["e2e"]["value"]), {k: round(x*1000,1) for k,x in r["stage_ms"].items()}, r["kernel"], round(r["frac"],3))
    except Exception as e: pass
PY
