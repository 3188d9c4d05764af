#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_head_gpu.py -q -x -rf > $OUT/pytest_head.log 2>&1; tail -15 $OUT/pytest_head.log
for q in 1 2 4 8; do
  SC_HEAD_CLUSTER=$q timeout 300 python bench.py --mode head --steps 30 --warmup 3 > $OUT/bench_head_q$q.json 2> $OUT/bench_head_q$q.err
  python -c "import json;d=json.load(open('$OUT/bench_head_q$q.json'));print($q, d['ms_per_step'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline']['tensor']['frac'], d['unfused']['ms_per_step'])" || tail -3 $OUT/bench_head_q$q.err
done
