#!/bin/bash
# r3e: head with CTA pairs + two tiles by default: the full head suite, large logits, compact head, sanitizer, bench.
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_head_gpu.py tests/test_parity_large_gpu.py tests/test_compact_gpu.py -q -m gpu -x --timeout 300 > $OUT/r3e_tests.log 2>&1; echo rc=$?; tail -2 $OUT/r3e_tests.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_kernels.py > $OUT/r3e_memcheck.log 2>&1; echo memcheck_rc=$?; tail -2 $OUT/r3e_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_kernels.py > $OUT/r3e_synccheck.log 2>&1; echo synccheck_rc=$?; tail -2 $OUT/r3e_synccheck.log
for i in 1 2; do
timeout 300 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r3e_head.json 2>&1
echo "head cfg2: $(python -c "import json;d=json.loads(open('$OUT/r3e_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
timeout 600 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r3e_head3.json 2>&1
echo "head cfg3: $(python -c "import json;d=json.loads(open('$OUT/r3e_head3.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
