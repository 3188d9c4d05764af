#!/bin/bash
# full-size parity tests + ncu captures of the multi-app TMA path (cfg4)
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
nproc
( time timeout 1200 python -m pytest tests/test_fullsize_gpu.py -x -q ) > $OUT/fullsize.log 2>&1; tail -4 $OUT/fullsize.log
for dt in bf16 f32; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 2 -c 1 \
      -o $OUT/prof_cfg4_${dt}_tma -f python bench.py --config 4 --dtype $dt --kernel tma --steps 2 --warmup 1 \
      --no-cpu-baseline --no-e2e > $OUT/ncu_cfg4_$dt.log 2>&1
  tail -1 $OUT/ncu_cfg4_$dt.log | cut -c1-200
done
