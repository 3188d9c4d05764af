#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_head_gpu.py -q -x -rf > $OUT/pytest_head.log 2>&1; tail -5 $OUT/pytest_head.log
for cfg in "SC_HEAD_PROBE=15" "SC_HEAD_PROBE=7" "SC_HEAD_PROBE=0" "SC_HEAD_X2D=1 SC_HEAD_PROBE=7" "SC_HEAD_KBS=2 SC_HEAD_PROBE=7" "SC_HEAD_KBS=2" "SC_HEAD_CLUSTER=1" "SC_HEAD_CLUSTER=4"; do
  env $cfg timeout 300 python bench.py --mode head --d 2048 --steps 20 --warmup 3 > $OUT/bh.json 2> $OUT/bh.err
  python -c "import json;d=json.load(open('$OUT/bh.json'));print('$cfg', d['roofline']['kernel'], 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'step_ms', round(d['ms_per_step'],4), 'unfused', round(d['unfused']['ms_per_step'],4))" || tail -3 $OUT/bh.err
done
