#!/bin/bash
# r3f: dense-gradient bench line, f32 and bf16.
OUT=gpurun_out
for dt in f32 bf16; do
timeout 600 python bench.py --grad dense --dtype $dt --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r3f_bench_dense_$dt.json 2>&1
echo "dense $dt: $(python -c "import json;d=json.loads(open('$OUT/r3f_bench_dense_$dt.json').read().strip().splitlines()[-1]);r=d['roofline'];print('%.4g'%d['value'], r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3), r['algorithmic_bytes_per_row'])" 2>&1 | tail -1)"
done
