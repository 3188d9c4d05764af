set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_parity_large_gpu.py tests/test_ranges_gpu.py -x -q -m gpu > gpurun_out/r2a_new_tests.log 2>&1; echo new_rc=$?
tail -30 gpurun_out/r2a_new_tests.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r2a_pytest_gpu.log 2>&1; echo all_rc=$?
tail -15 gpurun_out/r2a_pytest_gpu.log
SC_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_n2share.json 2> gpurun_out/r2a_bench_n2share.err; echo n2_rc=$?
tail -c 1500 gpurun_out/r2a_bench_n2share.json; tail -5 gpurun_out/r2a_bench_n2share.err
timeout 300 python bench.py --mode ranges --steps 50 --warmup 5 > gpurun_out/r2a_bench_ranges.json 2>&1; cat gpurun_out/r2a_bench_ranges.json
