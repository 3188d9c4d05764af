#!/bin/bash
# r2w: head drain probes: loads only (16), reduction only (32), neither (48), default.
OUT=gpurun_out
for m in "SC_HEAD_PROBE=0" "SC_HEAD_PROBE=16" "SC_HEAD_PROBE=32" "SC_HEAD_PROBE=48"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r2w_out.txt 2> $OUT/r2w_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
done
