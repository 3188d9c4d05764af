#!/bin/bash
# head bottleneck probes: full / no epilogue reduction / no MMA / neither, at d=2048 and d=512
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for d in 2048 512; do
for pr in 0 1 2 3; do
  SC_HEAD_PROBE=$pr timeout 300 python bench.py --mode head --d $d --steps 20 --warmup 3 > $OUT/bh.json 2> $OUT/bh.err
  python -c "import json;d=json.load(open('$OUT/bh.json'));print('d=$d probe=$pr', d['roofline']['kernel'], 'kernel_ms', round(d['roofline']['kernel_ms'],4))" || tail -3 $OUT/bh.err
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 1 -c 1 \
    -o $OUT/prof_head2 -f python bench.py --mode head --steps 2 --warmup 1 > $OUT/ncu_head2.log 2>&1
tail -1 $OUT/ncu_head2.log
