#!/bin/bash
# r5o: same-box A/B of the fused head (cfg2, d = 2048) between the session-start libsc and the final one.
OUT=gpurun_out
PKG=paper_2310_07240_b200
cp $PKG/libsc.so /tmp/libsc_new.so
for rnd in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then cp $PKG/libsc_ab_old.so $PKG/libsc.so; else cp /tmp/libsc_new.so $PKG/libsc.so; fi
    timeout 300 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r5o_${v}_$rnd.json 2>/dev/null
    echo "$v $rnd: $(tail -1 $OUT/r5o_${v}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), round(r.get('frac'),3))" 2>&1 | tail -1)"
  done
done
cp /tmp/libsc_new.so $PKG/libsc.so
