#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hist_kernel|weights_kernel" -s 4 -c 2 \
    -o $OUT/prof_hist -f python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $OUT/prof_hist.ncu-rep
