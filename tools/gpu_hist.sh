#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pt_hist.log 2>&1; tail -2 $OUT/pt_hist.log
for h in warp rows; do for dt in f32 bf16; do
  SC_HIST=$h timeout 300 python bench.py --dtype $dt --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$h $dt', round(d['ms_per_step']*1e3,1), 'us/step', d['phases_us'], f\"{d['value']:.4g}\")"
done; done
