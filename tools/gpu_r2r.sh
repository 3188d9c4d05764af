#!/bin/bash
# r2r: CTA pairs (double-buffered accumulators, half of W per CTA) with deeper W rings.
OUT=gpurun_out
for m in "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=8" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=10" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=12" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=8 SC_HEAD_KBS=1" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=10 SC_HEAD_KBS=1" "SC_HEAD_WSTAGES=4"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r2r_out.txt 2> $OUT/r2r_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
  env $m timeout 300 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2r_head.json 2>&1
  echo "   bench: $(python -c "import json;d=json.loads(open('$OUT/r2r_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))" 2>&1 | tail -1)"
done
