#!/bin/bash
# r2o: all-apps padding-class change (parity + bench), head benches cfg2 / cfg3 (final round-2 head code).
OUT=gpurun_out
timeout 900 python -m pytest tests/test_allapps_gpu.py tests/test_head_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2o_tests.log 2>&1; echo rc=$?; tail -3 $OUT/r2o_tests.log
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2o_bench_allapps.json 2>&1; tail -c 700 $OUT/r2o_bench_allapps.json
timeout 300 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2o_bench_head_cfg2.json 2>&1; tail -c 1500 $OUT/r2o_bench_head_cfg2.json
timeout 600 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2o_bench_head_cfg3.json 2>&1; tail -c 1500 $OUT/r2o_bench_head_cfg3.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 2 -c 1 -o $OUT/prof_r2o_head -f python bench.py --mode head --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2o_launches_head.csv python bench.py --mode head --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_r2o_head.ncu-rep $OUT/r2o_launches_head.csv $OUT/ncu_head_cfg2_d2048.json $OUT/r2o_head_cfg2_d2048.txt 1048576 head_kernel > /dev/null 2>&1
rm -f $OUT/prof_r2o_head.ncu-rep
