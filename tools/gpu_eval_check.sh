#!/bin/bash
# eval kernel change: GPU parity suite + bench (f32, bf16) + ncu time of the eval kernel
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > $OUT/bench_f32.json 2>$OUT/bench_f32.err; python -c "import json;d=json.load(open('$OUT/bench_f32.json'));print('f32', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline']['eval_kernel'])"
timeout 600 python bench.py --dtype bf16 --no-e2e --no-cpu-baseline > $OUT/bench_bf16.json 2>$OUT/bench_bf16.err; python -c "import json;d=json.load(open('$OUT/bench_bf16.json'));print('bf16', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline']['eval_kernel'])"
for e in "SC_EPL=1" "SC_EPL=0"; do
  env $e timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum.per_second --clock-control none -k regex:eval_kernel -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "gpu__time|dram__" | tail -2 | tr '\n' ' '; echo " <- $e"
done
