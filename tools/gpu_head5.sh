#!/bin/bash
# x-only streaming vs ring depth (16 KB stages of 128 rows x 128 B)
OUT=${OUT:-gpurun_out}
for st in 2 4 5 8 13; do
  SC_HEAD_CLUSTER=1 SC_HEAD_STAGES=$st SC_HEAD_PROBE=15 timeout 300 python bench.py --mode head --d 2048 --steps 20 --warmup 3 > $OUT/bh.json 2> $OUT/bh.err
  python -c "import json;d=json.load(open('$OUT/bh.json'));print('stages=$st x-only', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'TB/s', round(4.295/d['roofline']['kernel_ms'],2))" || tail -3 $OUT/bh.err
done
