#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for q in 1 2; do
for pr in 0 3 4 5 7; do
  SC_HEAD_CLUSTER=$q SC_HEAD_PROBE=$pr timeout 300 python bench.py --mode head --d 2048 --steps 20 --warmup 3 > $OUT/bh.json 2> $OUT/bh.err
  python -c "import json;d=json.load(open('$OUT/bh.json'));print('q=$q probe=$pr', d['roofline']['kernel'], 'kernel_ms', round(d['roofline']['kernel_ms'],4))" || tail -3 $OUT/bh.err
done
done
