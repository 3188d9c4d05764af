#!/bin/bash
# r2i: full GPU suite on the round-2 kernels, smoke, default bench + reference arm, CPU split, sampler ncu.
OUT=gpurun_out
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/r2i_pytest_gpu.log 2>&1; echo all_rc=$?
tail -8 $OUT/r2i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2i_smoke.log 2>&1; echo smoke_rc=$?; tail -2 $OUT/r2i_smoke.log
timeout 900 python bench.py > $OUT/r2i_bench.json 2> $OUT/r2i_bench.err; echo bench_rc=$?; tail -c 3000 $OUT/r2i_bench.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/r2i_bench_ref.json 2> $OUT/r2i_bench_ref.err; tail -c 800 $OUT/r2i_bench_ref.json
timeout 300 python bench.py --mode sample --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2i_bench_sample.json 2>&1; tail -c 600 $OUT/r2i_bench_sample.json
timeout 600 ncu --set full --clock-control none -k regex:"sample|scatter|draw|count|scan" -c 5 -o $OUT/prof_r2i_sample -f python bench.py --mode sample --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r2i_sample.ncu-rep --page raw --csv > $OUT/raw_r2i_sample.csv 2>/dev/null
rm -f $OUT/prof_r2i_sample.ncu-rep
timeout 1200 python tools/cpu_baseline_split.py $OUT/r2_cpu_baseline_split.json 65536 2048 > $OUT/r2i_cpu_split.log 2>&1; echo split_rc=$?; tail -6 $OUT/r2i_cpu_split.log | cut -c1-200
