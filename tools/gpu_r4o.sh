#!/bin/bash
# r4o: warp-per-32-rows GT pre-pass (hist_rows_kernel) + the per-list epilogue behind a call
# boundary (PAT 1): parity (step, full-size shards, patterns, multi-rank) + bench lines.
OUT=gpurun_out
TAG=${TAG:-r4o}
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_parity_patterns_gpu.py tests/test_multirank_gpu.py tests/test_sampler_gpu.py -q -m gpu --timeout 900 > $OUT/${TAG}_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/${TAG}_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_$i.json 2>/dev/null
done
timeout 300 python bench.py --order multi_select --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_multi_select.json 2>/dev/null
timeout 300 python bench.py --dtype bf16 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_bf16.json 2>/dev/null
for f in $OUT/${TAG}_bench_*.json; do
  echo "$f: $(tail -1 $f | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], 'ms/step', round(d.get('ms_per_step',0),4), 'frac', round(r.get('frac',0),3), r.get('kernel_ms'), r.get('eval_kernel'), r.get('phases_us', d.get('phases_us')))" 2>&1 | tail -1)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep hist_rows $OUT/${TAG}_launches.csv | head -3
