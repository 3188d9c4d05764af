#!/bin/bash
# r5i: GT pre-pass with the list bits in the shared table (one load + OR per label), 32-bit
# label loop: same-box A/B of the step against the previous library, then its parity tests.
OUT=gpurun_out
PKG=paper_2310_07240_b200
cp $PKG/libsc.so /tmp/libsc_new.so
for rnd in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then cp $PKG/libsc_ab_old.so $PKG/libsc.so; else cp /tmp/libsc_new.so $PKG/libsc.so; fi
    timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r5i_${v}_$rnd.json 2>/dev/null
    echo "$v $rnd: $(tail -1 $OUT/r5i_${v}_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), d.get('phases_us'))" 2>&1 | tail -1)"
  done
done
cp /tmp/libsc_new.so $PKG/libsc.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_parity_patterns_gpu.py tests/test_sampler_gpu.py -q -m gpu --timeout 600 > $OUT/r5i_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/r5i_pytest.log
