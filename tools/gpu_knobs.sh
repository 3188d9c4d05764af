#!/bin/bash
# knob sweep: "ENV=.. ENV2=..|bench args" cases in $CASES (newline separated)
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
while IFS='|' read -r envs args; do
  [ -z "$args" ] && continue
  r=$(env $envs timeout 300 python bench.py $args --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python3 -c "
import json,sys
try:
  d=json.loads(sys.argv[1]); r=d['roofline']
  print(f\"{sys.argv[2]:40s} {sys.argv[3]:40s} kernel {r['kernel_ms']*1e3:8.1f} us dense_frac {r['dense_frac']:.3f} {r['eval_kernel']}\")
except Exception as e: print(sys.argv[2], sys.argv[3], 'FAILED', e)
" "$r" "$envs" "$args"
done <<< "$CASES"
