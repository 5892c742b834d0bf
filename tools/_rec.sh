for w in gist1m sift1m; do
  start=$(date +%s)
  python bench.py --workload $w --no-cpu-baseline > gpurun_out/rec_$w.json 2>/dev/null
  end=$(date +%s)
  python -c "import json; d=json.load(open('gpurun_out/rec_$w.json')); print('$w', d['recall'], round(d['value']), $end-$start, 's')"
done
