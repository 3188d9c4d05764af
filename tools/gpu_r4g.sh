#!/bin/bash
# r4g: Multi-Select / per-list slot path (PAT 1) with padding keys 0xFF, offsets from keys,
# last-slot bitmask; parity of the per-list patterns + bench lines.
OUT=gpurun_out
TAG=${TAG:-r4g}
timeout 1200 python -m pytest tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_compact_gpu.py tests/test_multirank_gpu.py -q -m gpu --timeout 600 > $OUT/${TAG}_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/${TAG}_pytest.log
for o in multi_select app_choice; do
timeout 300 python bench.py --order $o --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_$o.json 2>/dev/null
SC_FORCE_SLOTS=1 timeout 300 python bench.py --order $o --config 4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_${o}_cfg4.json 2>/dev/null
done
for f in $OUT/${TAG}_bench_*.json; do
  echo "$f: $(tail -1 $f | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], 'ms/step', round(d.get('ms_per_step',0),4), 'frac', round(r.get('frac',0),3), r.get('kernel_ms'), r.get('eval_kernel'))" 2>&1 | tail -1)"
done
