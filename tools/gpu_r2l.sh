#!/bin/bash
# r2l: head drain in 32-column rounds (parity) + timeline probes isolating the MMA rate.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r2l_head_tests.log 2>&1; echo head_rc=$?; tail -3 $OUT/r2l_head_tests.log
for m in "SC_NOP=1" "SC_HEAD_PROBE=4" "SC_HEAD_PROBE=8" "SC_HEAD_PROBE=12" "SC_HEAD_PROBE=13" "SC_HEAD_PROBE=1"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r2l_out.txt 2> $OUT/r2l_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
done
timeout 300 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2l_head.json 2>&1
echo "head cfg2: $(python -c "import json;d=json.loads(open('$OUT/r2l_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
