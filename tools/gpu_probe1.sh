#!/bin/bash
# zero-copy probe + refreshed ncu of the default bench kernel (tma_ring_list) and bf16
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 300 python tools/zero_copy_probe.py 2 262144 > $OUT/zc2.log 2>&1; cat $OUT/zc2.log | tail -6
timeout 300 python tools/zero_copy_probe.py 3 32768 > $OUT/zc3.log 2>&1; cat $OUT/zc3.log | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1b.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|hist_kernel" -s 2 -c 2 \
    -o $OUT/prof_r1b -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_r1b.log 2>&1
tail -2 $OUT/ncu_r1b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 1 -c 1 \
    -o $OUT/prof_r1b_bf16 -f python bench.py --dtype bf16 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_r1b_bf16.log 2>&1
tail -2 $OUT/ncu_r1b_bf16.log
ls $OUT
