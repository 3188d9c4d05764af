set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_ranges_gpu.py -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --mode ranges --steps 100 --warmup 10 > gpurun_out/r2c_bench_ranges_new_$i.json 2>&1; cat gpurun_out/r2c_bench_ranges_new_$i.json; done
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/r2c_sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -5 gpurun_out/r2c_sanitizer_$tool.log
done
cp paper_2310_07240_b200/csrc/sc_ranges.cu /tmp/new_ranges.cu
cp tools/_old_sc_ranges.cu paper_2310_07240_b200/csrc/sc_ranges.cu
python -c "import sys; sys.path.insert(0,'.'); import importlib.util as u; s=u.spec_from_file_location('b','paper_2310_07240_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)"
for i in 1 2; do timeout 300 python bench.py --mode ranges --steps 100 --warmup 10 > gpurun_out/r2c_bench_ranges_old_$i.json 2>&1; cat gpurun_out/r2c_bench_ranges_old_$i.json; done
cp /tmp/new_ranges.cu paper_2310_07240_b200/csrc/sc_ranges.cu
