#!/bin/bash
# r3d: A/B lone two-tile head vs CTA pairs with two tiles, alternating, 3 rounds; d = 1024 / 2048.
OUT=gpurun_out
for d in 2048 1024; do for i in 1 2 3; do
  for m in "SC_NOP=1" "SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1"; do
    env $m timeout 300 python bench.py --mode head --d $d --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r3d_head.json 2>&1
    echo "d=$d [$m]: $(python -c "import json;d=json.loads(open('$OUT/r3d_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))" 2>&1 | tail -1)"
  done
done; done
