#!/bin/bash
# r2x: head with vote-uniform mbarrier waits in the MMA warp: parity + bench + trace.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r2x_head_tests.log 2>&1; echo rc=$?; tail -2 $OUT/r2x_head_tests.log
rm -f /tmp/trace.bin
SC_HEAD_TRACE=/tmp/trace.bin timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -1
for i in 1 2; do
timeout 300 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2x_head.json 2>&1
echo "head cfg2: $(python -c "import json;d=json.loads(open('$OUT/r2x_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
timeout 600 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2x_head3.json 2>&1
echo "head cfg3: $(python -c "import json;d=json.loads(open('$OUT/r2x_head3.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
