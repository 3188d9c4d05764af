#!/bin/bash
# r3b: CTA-pair head timeline incl. the peer CTA's producers.
OUT=gpurun_out
for m in "SC_HEAD_CLUSTER=2" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=8" "SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r3b_out.txt 2> $OUT/r3b_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -9
done
