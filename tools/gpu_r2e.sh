#!/bin/bash
# r2e: head under every pattern + column passes; compacted cfg3 bench; head benches cfg2 / cfg3.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x > $OUT/r2e_head_tests.log 2>&1; echo head_rc=$?
tail -15 $OUT/r2e_head_tests.log
timeout 600 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2e_bench_head_cfg2.json 2> $OUT/r2e_bench_head_cfg2.err; tail -c 1500 $OUT/r2e_bench_head_cfg2.json; tail -3 $OUT/r2e_bench_head_cfg2.err
timeout 900 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2e_bench_head_cfg3.json 2> $OUT/r2e_bench_head_cfg3.err; tail -c 1500 $OUT/r2e_bench_head_cfg3.json; tail -3 $OUT/r2e_bench_head_cfg3.err
timeout 900 python bench.py --config 3 --compact --steps 50 --warmup 5 --no-cpu-baseline > $OUT/r2e_bench_cfg3_compact.json 2> $OUT/r2e_bench_cfg3_compact.err; tail -c 2500 $OUT/r2e_bench_cfg3_compact.json; tail -3 $OUT/r2e_bench_cfg3_compact.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2e_bench_cfg3_dense.json 2> $OUT/r2e_bench_cfg3_dense.err; tail -c 1500 $OUT/r2e_bench_cfg3_dense.json; tail -3 $OUT/r2e_bench_cfg3_dense.err
