#!/bin/bash
# r2p: sampler with the parallel stable scatter (parity + bench + launch times).
OUT=gpurun_out
timeout 600 python -m pytest tests/test_sampler_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2p_tests.log 2>&1; echo rc=$?; tail -3 $OUT/r2p_tests.log
timeout 300 python bench.py --mode sample --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r2p_bench_sample.json 2>&1; tail -c 700 $OUT/r2p_bench_sample.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/r2p_sampler_launches.csv python bench.py --mode sample --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "kernel" $OUT/r2p_sampler_launches.csv | grep -E "count|scan|starts|scatter|draw" | tail -15 | cut -c1-220
