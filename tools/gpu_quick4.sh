#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
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
B="timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
for fl in 0 1 2 3; do
line "cfg3 f32 gather flavor $fl"   SC_LD_FLAVOR=$fl $B --config 3 --kernel gather
line "cfg2 f32 gather flavor $fl"   SC_LD_FLAVOR=$fl $B --kernel gather
done
SC_LD_FLAVOR=1 timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum -k regex:"gather_kernel" -s 2 -c 1 python bench.py --config 3 --kernel gather --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "dram__|lts__|gpu__"
