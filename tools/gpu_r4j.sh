#!/bin/bash
# r4j: ncu full capture of the all-apps lane-per-row kernel (cfg4, 2^18 rows).
OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"all_apps" -s 1 -c 1 -o $OUT/prof_r4j -f python bench.py --mode all_apps --config 4 --rows 262144 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r4j.ncu-rep --page raw --csv > $OUT/raw_r4j.csv 2>/dev/null
ncu -i $OUT/prof_r4j.ncu-rep --page source --csv --print-source sass > $OUT/src_r4j.csv 2>/dev/null
ncu -i $OUT/prof_r4j.ncu-rep --page details > $OUT/det_r4j.txt 2>/dev/null
rm -f $OUT/prof_r4j.ncu-rep
ls -la $OUT/*r4j*
