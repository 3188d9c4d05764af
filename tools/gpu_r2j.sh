#!/bin/bash
# r2j: head timeline probe at d = 512 / 2048 (cfg2), default and one-tile mode.
OUT=gpurun_out
for cfg in "2048 x" "512 x" "2048 SC_HEAD_T2=0"; do set -- $cfg
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin ${2/x/SC_NOP=1} timeout 300 python bench.py --mode head --d $1 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2> $OUT/r2j_err.txt
  echo "== d=$1 $2"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -12
done
