#!/bin/bash
# NEXT f4 evidence: parity tests, bench lines (d=2048, d=512), launch list + ncu full capture
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_head_gpu.py -q -rf > $OUT/pytest_head.log 2>&1; tail -3 $OUT/pytest_head.log
timeout 600 python bench.py --mode head --steps 50 --warmup 5 > $OUT/bench_head.json 2> $OUT/bench_head.err; tail -1 $OUT/bench_head.json
timeout 600 python bench.py --mode head --d 512 --steps 50 --warmup 5 > $OUT/bench_head_d512.json 2> $OUT/bench_head_d512.err; tail -1 $OUT/bench_head_d512.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_head.csv \
    python bench.py --mode head --steps 3 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 1 -c 1 \
    -o $OUT/prof_head -f python bench.py --mode head --steps 2 --warmup 1 > $OUT/ncu_head.log 2>&1
tail -1 $OUT/ncu_head.log
