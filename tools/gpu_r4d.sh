#!/bin/bash
# r4d: ncu full capture of the Multi-Select eval kernel (cfg2 f32) and the value-ranges kernels.
OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_r4d_ms -f python bench.py --order multi_select --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r4d_ms.ncu-rep --page raw --csv > $OUT/raw_r4d_ms.csv 2>/dev/null
ncu -i $OUT/prof_r4d_ms.ncu-rep --page source --csv --print-source sass > $OUT/src_r4d_ms.csv 2>/dev/null
ncu -i $OUT/prof_r4d_ms.ncu-rep --page details > $OUT/det_r4d_ms.txt 2>/dev/null
rm -f $OUT/prof_r4d_ms.ncu-rep
ls -la $OUT/*r4d*
