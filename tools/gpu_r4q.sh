#!/bin/bash
# r4q: dense-gradient deferral as its own instantiation (eval_kernel<..., DEFER>): same-box A/B
# against the session-start libsc (f32 / bf16 sparse-gradient lines), the dense lines, and the
# dense-gradient parity tests.
OUT=gpurun_out
PKG=paper_2310_07240_b200
cp $PKG/libsc.so /tmp/libsc_new.so
for rnd in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp $PKG/libsc_ab_old.so $PKG/libsc.so; else cp /tmp/libsc_new.so $PKG/libsc.so; fi
    for a in "f32:" "bf16:--dtype bf16" "densef32:--grad dense" "densebf16:--grad dense --dtype bf16"; do
      n=${a%%:*}; args=${a#*:}
      timeout 300 python bench.py $args --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r4q_${v}_${n}_$rnd.json 2>/dev/null
      echo "$v $n $rnd: $(tail -1 $OUT/r4q_${v}_${n}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print(round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), round(r.get('frac'),3))" 2>&1 | tail -1)"
    done
  done
done
cp /tmp/libsc_new.so $PKG/libsc.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_patterns_gpu.py tests/test_parity_large_gpu.py tests/test_compact_gpu.py -q -m gpu --timeout 600 > $OUT/r4q_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/r4q_pytest.log
