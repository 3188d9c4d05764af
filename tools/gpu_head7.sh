#!/bin/bash
OUT=${OUT:-gpurun_out}
for cfg in "SC_HEAD_PROBE=39 SC_HEAD_KBS=4" "SC_HEAD_PROBE=103 SC_HEAD_KBS=4" "SC_HEAD_PROBE=103 SC_HEAD_KBS=1" "SC_HEAD_PROBE=103 SC_HEAD_KBS=4 SC_HEAD_CLUSTER=1" "SC_HEAD_PROBE=39 SC_HEAD_KBS=4 SC_HEAD_CLUSTER=1" "SC_HEAD_PROBE=119 SC_HEAD_KBS=4 SC_HEAD_CLUSTER=1"; do
  env $cfg timeout 300 python bench.py --mode head --d 2048 --steps 20 --warmup 3 > $OUT/bh.json 2> $OUT/bh.err
  python -c "import json;d=json.load(open('$OUT/bh.json'));print('$cfg', d['roofline']['kernel'], 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'TB/s', round(4.295/d['roofline']['kernel_ms'],2))" || tail -3 $OUT/bh.err
done
