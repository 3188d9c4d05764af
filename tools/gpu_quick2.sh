#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
SC_BLOCKED=1 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "configs and tma" 2>&1 | tail -2
line() {
  local label="$1"; shift
  env "$@" > $OUT/q.json 2>$OUT/q.err
  python - "$OUT/q.json" "$label" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:44s} {d['value']:.3e}/s kernel {r['kernel_ms']*1e3:7.1f} us dense_frac {r['dense_frac']:.3f} frac {r['frac']:.3f} step {d['ms_per_step']*1e3:7.1f} us {r['eval_kernel']}")
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
}
B="timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e"
line "f32 default"                 $B
line "f32 blocked"                 SC_BLOCKED=1 $B
line "f32 blocked NG1 64K"         SC_BLOCKED=1 SC_NG=1 SC_STAGE_KB=64 $B
line "f32 EPL0 blocked"            SC_BLOCKED=1 SC_EPL=0 $B
line "bf16 NG2 32K"                SC_NG=2 SC_STAGE_KB=32 $B --dtype bf16
line "bf16 NG2 32K blocked"        SC_BLOCKED=1 SC_NG=2 SC_STAGE_KB=32 $B --dtype bf16
line "cfg3 f32 tma blocked"        SC_BLOCKED=1 $B --config 3 --kernel tma
line "cfg3 f32 tma"                $B --config 3 --kernel tma
