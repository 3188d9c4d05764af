#!/bin/bash
# r5m: pipeline-shape knobs on the dense-gradient (DEFER) and column-compacted (dense-mapped) paths.
OUT=gpurun_out
run() { local name=$1; shift
  env "$@" timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $ARGS > $OUT/r5m_$name.json 2>/dev/null
  echo "$name: $(tail -1 $OUT/r5m_$name.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(r.get('kernel_ms'),4), 'frac', round(r.get('frac',0),3), r.get('eval_kernel'))" 2>&1 | tail -1)"
}
for cfg in "dense:--grad dense" "densebf:--grad dense --dtype bf16" "c3c:--config 3 --compact" "c3cbf:--config 3 --compact --dtype bf16"; do
  n=${cfg%%:*}; ARGS=${cfg#*:}
  run ${n}_base X=1
  run ${n}_ng2_32 SC_NG=2 SC_STAGE_KB=32
  run ${n}_ng1_32 SC_NG=1 SC_STAGE_KB=32
  run ${n}_ng4_16 SC_NG=4 SC_STAGE_KB=16
done
