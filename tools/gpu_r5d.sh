#!/bin/bash
# r5d: GT pre-pass with four rows per thread (loads in flight together): parity + step timing.
OUT=gpurun_out
for rnd in 1 2 3; do
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r5d_$rnd.json 2>/dev/null
  echo "$rnd: $(tail -1 $OUT/r5d_$rnd.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], round(d.get('ms_per_step',0),4), round(r.get('kernel_ms'),4), d.get('phases_us'))" 2>&1 | tail -1)"
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_multirank_gpu.py tests/test_sampler_gpu.py -q -m gpu --timeout 600 > $OUT/r5d_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/r5d_pytest.log
