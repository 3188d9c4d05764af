#!/bin/bash
# r2m: MMA column chunks as independent accumulator chains: parity + timing sweep.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r2m_head_tests.log 2>&1; echo head_rc=$?; tail -3 $OUT/r2m_head_tests.log
for m in "SC_HEAD_NCHUNK=1" "SC_HEAD_NCHUNK=2" "SC_HEAD_NCHUNK=1 SC_HEAD_T2=0" "SC_HEAD_NCHUNK=1 SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1" "SC_HEAD_NCHUNK=1 SC_HEAD_CLUSTER=2" "SC_HEAD_PROBE=12"; do
  rm -f /tmp/trace.bin
  env SC_HEAD_TRACE=/tmp/trace.bin $m timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/r2m_out.txt 2> $OUT/r2m_err.txt
  echo "== $m"; python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
  env $m timeout 300 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2m_head.json 2>&1
  echo "   bench: $(python -c "import json;d=json.loads(open('$OUT/r2m_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
for m in "SC_HEAD_NCHUNK=1" "SC_HEAD_NCHUNK=2"; do
  env $m timeout 600 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2m_head3.json 2>&1
  echo "cfg3 head [$m]: $(python -c "import json;d=json.loads(open('$OUT/r2m_head3.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
