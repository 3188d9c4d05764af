#!/bin/bash
# r5e: sigma and its derivative from one exponential and one division in every epilogue
# (sig_dsig_f): same-box A/B against the previous commit (libsc_ab_old.so), then the full GPU suite.
OUT=gpurun_out
PKG=paper_2310_07240_b200
cp $PKG/libsc.so /tmp/libsc_new.so
for rnd in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp $PKG/libsc_ab_old.so $PKG/libsc.so; else cp /tmp/libsc_new.so $PKG/libsc.so; fi
    for a in "f32:" "bf16:--dtype bf16" "ms:--order multi_select" "ac:--order app_choice" "head:--mode head --steps 50" "dense:--grad dense --steps 50"; do
      n=${a%%:*}; args=${a#*:}
      timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e $args > $OUT/r5e_${v}_${n}_$rnd.json 2>/dev/null
      echo "$v $n $rnd: $(tail -1 $OUT/r5e_${v}_${n}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), round(r.get('frac'),3))" 2>&1 | tail -1)"
    done
  done
done
cp /tmp/libsc_new.so $PKG/libsc.so
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/r5e_pytest_gpu.log 2>&1; echo all_rc=$?; tail -2 $OUT/r5e_pytest_gpu.log
