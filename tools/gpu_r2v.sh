#!/bin/bash
# r2v: per-list patterns with lane-folded slots (one warp arg max per list): parity + bench.
OUT=gpurun_out
timeout 1500 python -m pytest tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_multirank_gpu.py tests/test_compact_gpu.py -q -m gpu -x --timeout 600 > $OUT/r2v_tests.log 2>&1; echo rc=$?; tail -3 $OUT/r2v_tests.log
SC_AC2=0 timeout 1500 python -m pytest tests/test_parity_patterns_gpu.py -q -m gpu -x --timeout 600 > $OUT/r2v_tests_slots.log 2>&1; echo rc_slots=$?; tail -2 $OUT/r2v_tests_slots.log
for o in multi_select; do for dt in f32 bf16; do
  timeout 300 python bench.py --config 2 --dtype $dt --order $o --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2v_${o}_$dt.json 2>&1
  echo "$o $dt: $(python -c "import json;d=json.loads(open('$OUT/r2v_${o}_$dt.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3),'%.4g'%d['value'])")"
done; done
SC_AC2=0 timeout 300 python bench.py --config 2 --order app_choice --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2v_ac_slots.json 2>&1
echo "app-choice slots: $(python -c "import json;d=json.loads(open('$OUT/r2v_ac_slots.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3),'%.4g'%d['value'])")"
