#!/bin/bash
# r5l: the slot path (Multi-Select) on two warp groups by default: bench + per-list parity.
OUT=gpurun_out
for rnd in 1 2; do
for a in "ms:--order multi_select" "ms_cfg4:--order multi_select --config 4 --steps 30" "ms_bf16:--order multi_select --dtype bf16"; do
  n=${a%%:*}; args=${a#*:}
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $args > $OUT/r5l_${n}_$rnd.json 2>/dev/null
  echo "$n $rnd: $(tail -1 $OUT/r5l_${n}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), round(r.get('frac'),3))" 2>&1 | tail -1)"
done
done
timeout 900 python -m pytest tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_compact_gpu.py tests/test_multirank_gpu.py -q -m gpu --timeout 600 > $OUT/r5l_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/r5l_pytest.log
