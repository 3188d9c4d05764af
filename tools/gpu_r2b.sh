set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_large_gpu.py tests/test_ranges_gpu.py tests/test_parity_gpu.py -q -m gpu -x > gpurun_out/r2b_new_tests.log 2>&1; echo new_rc=$?
tail -30 gpurun_out/r2b_new_tests.log
for i in 1 2; do timeout 300 python bench.py --mode ranges --steps 100 --warmup 10 > gpurun_out/r2b_bench_ranges_$i.json 2>&1; cat gpurun_out/r2b_bench_ranges_$i.json; done
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2b_bench.json 2>&1; tail -c 1200 gpurun_out/r2b_bench.json
