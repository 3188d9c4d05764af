#!/bin/bash
# One GPU round: parity tests, the bench matrix, and ncu captures of chosen configs.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
bash tools/gpu_bench_matrix.sh 2>&1 | tee $OUT/matrix.txt
# ncu captures: "config dtype kernel" triples in $NCU_CASES
for c in ${NCU_CASES:-}; do
  IFS=: read cfg dt k <<< "$c"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|gather_kernel" -s 2 -c 1 \
      -o $OUT/prof_cfg${cfg}_${dt}_${k} -f python bench.py --config $cfg --dtype $dt --kernel $k --steps 2 --warmup 1 \
      --no-cpu-baseline --no-e2e > $OUT/ncu_cfg${cfg}_${dt}_${k}.log 2>&1
  tail -1 $OUT/ncu_cfg${cfg}_${dt}_${k}.log
done
