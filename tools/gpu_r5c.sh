#!/bin/bash
# r5c: GT pre-pass grid size (CTAs per SM) against its 18.8 us in the step.
OUT=gpurun_out
for rnd in 1 2; do
for g in 8 4 2 1 16; do
  SC_HIST_CTAS_PER_SM=$g timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r5c_g${g}_$rnd.json 2>/dev/null
  echo "g=$g $rnd: $(tail -1 $OUT/r5c_g${g}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), d.get('phases_us'))" 2>&1 | tail -1)"
done
done
