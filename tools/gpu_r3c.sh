#!/bin/bash
# r3c: CTA pairs with the leader expecting both CTAs' bytes: parity + trace + bench.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r3c_head_tests.log 2>&1; echo rc=$?; tail -2 $OUT/r3c_head_tests.log
for m in "SC_HEAD_CLUSTER=2" "SC_HEAD_CLUSTER=2 SC_HEAD_WSTAGES=8" "SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1" "SC_NOP=1"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r3c_out.txt 2> $OUT/r3c_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
  env $m timeout 300 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r3c_head.json 2>&1
  echo "   bench: $(python -c "import json;d=json.loads(open('$OUT/r3c_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))" 2>&1 | tail -1)"
done
