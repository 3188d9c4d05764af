#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
line() {
  local label="$1"; shift
  env "$@" > $OUT/q.json 2>$OUT/q.err
  python - "$OUT/q.json" "$label" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:30s} {d['value']:.3e}/s kernel {r['kernel_ms']*1e3:7.1f} us dense_frac {r['dense_frac']:.3f} frac {r['frac']:.3f} step {d['ms_per_step']*1e3:7.1f} us {r['eval_kernel']} {d.get('phases_us')}")
except Exception as e: print(sys.argv[2], "FAILED", e, open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
}
B="timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e"
line "f32 default"                 $B
line "bf16 default"                $B --dtype bf16
line "cfg4 default"                $B --config 4
