#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for dt in f32 bf16; do
for cfgs in "SC_NG=1 SC_STAGE_KB=64" "SC_NG=1 SC_STAGE_KB=64 SC_SPLIT_COPY=1" "SC_NG=1 SC_STAGE_KB=64 SC_NO_EVICT_FIRST=1" "SC_EPL=0" "SC_EPL=0 SC_SPLIT_COPY=1" "SC_EPL=0 SC_NO_EVICT_FIRST=1" "SC_EPL=0 SC_STAGE_KB=32"; do
  env $cfgs timeout 300 python bench.py --config 2 --dtype $dt --kernel tma --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/sw.json 2>/dev/null
  python - "$OUT/sw.json" "$dt $cfgs" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:50s} kernel {r['kernel_ms']*1e3:7.1f} us  dense_frac {r['dense_frac']:.3f}  step {d['ms_per_step']*1e3:7.1f} us")
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
done; done
SC_NG=1 SC_STAGE_KB=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 2 -c 1 \
      -o $OUT/prof_bf16_ng1 -f python bench.py --config 2 --dtype bf16 --kernel tma --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
SC_EPL=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 2 -c 1 \
      -o $OUT/prof_f32_epl0 -f python bench.py --config 2 --dtype f32 --kernel tma --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $OUT/*.ncu-rep
