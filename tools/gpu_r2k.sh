#!/bin/bash
# r2k: head timeline probe for CTA pairs (one / two row tiles) at d = 2048.
OUT=gpurun_out
for m in "SC_HEAD_CLUSTER=2" "SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r2k_out.txt 2> $OUT/r2k_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -7
done
