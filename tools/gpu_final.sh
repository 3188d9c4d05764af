#!/bin/bash
# bench line (default config) + ncu launch list + ncu full capture of the eval kernel, for profiles/
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1}
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $OUT/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
kill $SMI
tail -1 $OUT/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
tail -1 $OUT/bench_ref_$TAG.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|gather_kernel" -s 2 -c 1 \
    -o $OUT/prof_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for dt in bf16; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|gather_kernel" -s 2 -c 1 \
      -o $OUT/prof_${TAG}_$dt -f python bench.py --dtype $dt --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
ls $OUT/*.ncu-rep
