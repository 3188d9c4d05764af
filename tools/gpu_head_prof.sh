#!/bin/bash
# head kernel: bench line (single CTA / CTA pair) + ncu full capture of each
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for pc in 1 2; do
  SC_HEAD_CLUSTER=$pc timeout 300 python bench.py --mode head --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-600
  SC_HEAD_CLUSTER=$pc timeout 600 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 2 -c 1 \
      -o $OUT/prof_head_c$pc -f python bench.py --mode head --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_head_c$pc.log 2>&1
  tail -1 $OUT/ncu_head_c$pc.log
done
