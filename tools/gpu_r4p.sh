#!/bin/bash
# r4p: same-box A/B of libsc at the session start (8f754fb, libsc_ab_old.so) against the
# working tree (dense-gradient drain, slot path, hist pre-pass, per-list epilogue call):
# f32 / bf16 / Multi-Select bench lines, interleaved; then the r4o parity run on the new lib.
OUT=gpurun_out
PKG=paper_2310_07240_b200
cp $PKG/libsc.so /tmp/libsc_new.so
for rnd in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp $PKG/libsc_ab_old.so $PKG/libsc.so; else cp /tmp/libsc_new.so $PKG/libsc.so; fi
    for a in "f32:" "bf16:--dtype bf16" "ms:--order multi_select"; do
      n=${a%%:*}; args=${a#*:}
      timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r4p_${v}_${n}_$rnd.json 2>/dev/null
      echo "$v $n $rnd: $(tail -1 $OUT/r4p_${v}_${n}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), d.get('phases_us'))" 2>&1 | tail -1)"
    done
  done
done
cp /tmp/libsc_new.so $PKG/libsc.so
bash tools/gpu_r4o.sh
