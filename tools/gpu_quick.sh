#!/bin/bash
# parity + a few targeted bench lines (run on the GPU box)
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
line() {  # label, env..., -- bench args
  local label="$1"; shift
  env "$@" > $OUT/q.json 2>$OUT/q.err
  python - "$OUT/q.json" "$label" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:44s} {d['value']:.3e}/s kernel {r['kernel_ms']*1e3:7.1f} us dense_frac {r['dense_frac']:.3f} frac {r['frac']:.3f} step {d['ms_per_step']*1e3:7.1f} us {r['eval_kernel']}")
except Exception as e: print(sys.argv[2], "FAILED", e, open(sys.argv[1].replace('.json','.err')).read()[-500:])
PY
}
B="timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e"
line "f32 1M default"            $B
line "f32 4M rows"               $B --rows 4194304
line "f32 4M rows EPL0"          SC_EPL=0 $B --rows 4194304
line "bf16 1M default"           $B --dtype bf16
line "bf16 1M NG2 32K"           SC_NG=2 SC_STAGE_KB=32 $B --dtype bf16
line "bf16 4M"                   $B --dtype bf16 --rows 4194304
