#!/bin/bash
# Sweep eval-kernel pipeline shapes on cfg2 (run on the GPU box).
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for dt in f32 bf16; do
for cfgs in "SC_NG=1 SC_STAGE_KB=64" "SC_NG=1 SC_STAGE_KB=32" "SC_NG=2 SC_STAGE_KB=32" "SC_NG=2 SC_STAGE_KB=16" "SC_NG=4 SC_STAGE_KB=16" "SC_NG=4 SC_STAGE_KB=8" "SC_NG=8 SC_STAGE_KB=8" "SC_EPL=0"; do
  env $cfgs timeout 300 python bench.py --config 2 --dtype $dt --kernel tma --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/sw.json 2>/dev/null
  python - "$OUT/sw.json" "$dt $cfgs" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:36s} kernel {r['kernel_ms']*1e3:7.1f} us  dense_frac {r['dense_frac']:.3f}  step {d['ms_per_step']*1e3:7.1f} us")
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
done; done
