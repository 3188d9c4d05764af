#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
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
line "bf16 default"                $B --dtype bf16
line "f32 gather L2fetch32"        SC_L2_FETCH=32 $B --kernel gather
line "f32 gather L2fetch64"        SC_L2_FETCH=64 $B --kernel gather
line "cfg3 f32 gather L2fetch32"   SC_L2_FETCH=32 $B --config 3 --kernel gather
line "cfg3 f32 gather"             $B --config 3 --kernel gather
SC_L2_FETCH=32 timeout 600 ncu --set full --clock-control none -k regex:"gather_kernel" -s 2 -c 1 \
      -o $OUT/prof_cfg3_gather_l2f32 -f python bench.py --config 3 --kernel gather --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $OUT/*.ncu-rep
