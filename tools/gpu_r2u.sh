#!/bin/bash
# r2u: application-choice order by two arg maxima (pat 3): parity (patterns, large logits,
# multi-rank, compact, fullsize) + bench vs the slot path.
OUT=gpurun_out
timeout 1500 python -m pytest tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_multirank_gpu.py tests/test_compact_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -m gpu -x --timeout 600 > $OUT/r2u_tests.log 2>&1; echo rc=$?; tail -3 $OUT/r2u_tests.log
for m in "SC_NOP=1" "SC_AC2=0"; do
  for dt in f32 bf16; do
    env $m timeout 300 python bench.py --config 2 --dtype $dt --order app_choice --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2u_ac.json 2>&1
    echo "app-choice $dt [$m]: $(python -c "import json;d=json.loads(open('$OUT/r2u_ac.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3),'%.4g'%d['value'])")"
    cp $OUT/r2u_ac.json $OUT/r2u_ac_${dt}_$(echo $m | tr '=' '_').json
  done
done
timeout 300 python bench.py --config 4 --order app_choice --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2u_ac_cfg4.json 2>&1
echo "app-choice cfg4: $(python -c "import json;d=json.loads(open('$OUT/r2u_ac_cfg4.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3),'%.4g'%d['value'])")"
