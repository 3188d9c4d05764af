#!/bin/bash
OUT=${OUT:-gpurun_out}
SC_HEAD_PROBE=127 SC_HEAD_KBS=4 SC_HEAD_CLUSTER=1 timeout 600 ncu --set full --clock-control none -k regex:"head_kernel" -c 1 -o $OUT/prof_headx -f python bench.py --mode head --d 2048 --steps 1 --warmup 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"probe" -s 2 -c 1 -o $OUT/prof_stream -f ./tools/stream_probe.bin 1 > /dev/null 2>&1
ls $OUT/*.ncu-rep
