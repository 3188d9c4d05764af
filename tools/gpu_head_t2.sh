#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_head_gpu.py -x -q > $OUT/pt_head.log 2>&1; tail -3 $OUT/pt_head.log
run() {
  echo "$1 d=$2"; env $1 timeout 300 python bench.py --mode head --d $2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "
import json,sys
l=sys.stdin.read().strip()
try:
  d=json.loads(l); r=d['roofline']; print(f\"  step {d['ms_per_step']:.3f} ms kernel {r['kernel_ms']:.3f} ms frac {r['frac']:.3f} unfused {d['unfused']['ms_per_step']:.3f}\")
except Exception as e: print('  FAILED', l[-300:])
"
}
for cfg in ${HEAD_CASES:-"SC_HEAD_T2=0:2048" "SC_HEAD_T2=1:2048"}; do run "${cfg%%:*}" "${cfg##*:}"; done
