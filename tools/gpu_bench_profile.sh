#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list, one full ncu capture of eval_kernel.
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
DT=${DT:-f32}
timeout 900 python bench.py --steps ${STEPS:-200} --warmup ${WARMUP:-10} --dtype $DT > $OUT/bench_$DT.json 2> $OUT/bench_$DT.err
tail -2 $OUT/bench_$DT.err
cat $OUT/bench_$DT.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$DT.csv \
      python bench.py --steps 3 --warmup 1 --dtype $DT --no-cpu-baseline --no-e2e > $OUT/ncu_launch_run.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 2 -c 1 \
      -o $OUT/prof_eval_$DT -f python bench.py --steps 2 --warmup 1 --dtype $DT --no-cpu-baseline --no-e2e > $OUT/ncu_full_run.log 2>&1
  tail -3 $OUT/ncu_full_run.log
fi
