#!/bin/bash
# r4b: dense gradient rows parked per warp and written between stages (not one 32-row burst per
# batch): parity of every dense-gradient test + the default and dense bench lines.
OUT=gpurun_out
TAG=${TAG:-r4b}
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_compact_gpu.py -q -m gpu --timeout 600 > $OUT/${TAG}_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/${TAG}_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_$i.json 2>/dev/null
timeout 300 python bench.py --grad dense --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_dense_f32_$i.json 2>/dev/null
timeout 300 python bench.py --grad dense --dtype bf16 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_dense_bf16_$i.json 2>/dev/null
done
timeout 300 python bench.py --grad dense --order app_choice --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_dense_appchoice.json 2>/dev/null
for f in $OUT/${TAG}_bench_*.json; do
  echo "$f: $(tail -1 $f | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], 'ms/step', round(d.get('ms_per_step',0),4), 'frac', round(r.get('frac',0),3), r.get('kernel_ms'))" 2>&1 | tail -1)"
done
