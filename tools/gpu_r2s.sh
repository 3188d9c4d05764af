#!/bin/bash
# r2s: all-apps keys with one-hot list bits (parity + bench).
OUT=gpurun_out
timeout 900 python -m pytest tests/test_allapps_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2s_tests.log 2>&1; echo rc=$?; tail -2 $OUT/r2s_tests.log
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2s_bench_allapps.json 2>&1; tail -c 700 $OUT/r2s_bench_allapps.json
timeout 600 python bench.py --mode all_apps --config 4 --dtype bf16 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2s_bench_allapps_bf16.json 2>&1; tail -c 300 $OUT/r2s_bench_allapps_bf16.json
