#!/bin/bash
# r5k: pipeline-shape knobs on the issue-bound variants (Multi-Select f32, app-choice f32, bf16 API order).
OUT=gpurun_out
run() { # name env... -- args
  local name=$1; shift
  env "$@" timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $ARGS > $OUT/r5k_$name.json 2>/dev/null
  echo "$name: $(tail -1 $OUT/r5k_$name.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(r.get('kernel_ms'),4), 'frac', round(r.get('frac',0),3), r.get('eval_kernel'))" 2>&1 | tail -1)"
}
for cfg in "ms:--order multi_select" "ac:--order app_choice" "bf:--dtype bf16" "api:"; do
  n=${cfg%%:*}; ARGS=${cfg#*:}
  run ${n}_base X=1
  run ${n}_ng4_48 SC_NG=4 SC_STAGE_KB=48
  run ${n}_ng2_32 SC_NG=2 SC_STAGE_KB=32
  run ${n}_ng2_48 SC_NG=2 SC_STAGE_KB=48
  run ${n}_ng1_32 SC_NG=1 SC_STAGE_KB=32
done
