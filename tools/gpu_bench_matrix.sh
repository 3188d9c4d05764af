#!/bin/bash
# Bench matrix for kernel selection (run on the GPU box).
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for args in "--config 2 --dtype f32 --kernel tma" "--config 2 --dtype f32 --kernel gather" \
            "--config 2 --dtype bf16 --kernel tma" "--config 2 --dtype bf16 --kernel gather" \
            "--config 3 --dtype f32 --kernel tma" "--config 3 --dtype f32 --kernel gather" \
            "--config 3 --dtype bf16 --kernel tma" "--config 3 --dtype bf16 --kernel gather" \
            "--config 4 --dtype f32 --kernel tma" "--config 4 --dtype f32 --kernel gather" \
            "--config 4 --dtype bf16 --kernel tma" "--config 4 --dtype bf16 --kernel gather" \
            "--config 5 --dtype f32" "--config 5 --dtype bf16" \
            "--config 1 --dtype f32 --kernel tma" "--config 1 --dtype f32 --kernel gather" \
            "--config 2 --dtype f32 --order app_choice" "--config 2 --dtype f32 --order multi_select"; do
  tag=$(echo $args | tr -d ' -' )
  timeout 300 python bench.py $args --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e > $OUT/m_$tag.json 2> $OUT/m_$tag.err
  python - "$OUT/m_$tag.json" "$args" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d["roofline"]
    print(f"{sys.argv[2]:40s} {d['value']:.3e} rows/s  step {d['ms_per_step']*1e3:8.1f} us  kernel {r['kernel_ms']*1e3:8.1f} us  frac {r['frac']:.3f}  dense_frac {r['dense_frac']:.3f}  {r['eval_kernel']}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
