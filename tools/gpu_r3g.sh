#!/bin/bash
# r3g: ncu of the eval kernel with the dense gradient (f32).
OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_r3g_dense -f python bench.py --grad dense --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r3g_dense.ncu-rep --page raw --csv > $OUT/raw_r3g_dense.csv 2>/dev/null
ncu -i $OUT/prof_r3g_dense.ncu-rep --page source --csv --print-source sass > $OUT/src_r3g_dense.csv 2>/dev/null
rm -f $OUT/prof_r3g_dense.ncu-rep
ls -la $OUT/raw_r3g_dense.csv $OUT/src_r3g_dense.csv
