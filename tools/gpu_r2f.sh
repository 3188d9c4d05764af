#!/bin/bash
# r2f: head tests (column passes fixed), host-entry tests, cfg3-compact kernel knobs, head pair/two-tile, head cfg3.
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r2f_head_tests.log 2>&1; echo head_rc=$?
tail -15 $OUT/r2f_head_tests.log
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x --timeout 240 -k "host" > $OUT/r2f_host_tests.log 2>&1; echo host_rc=$?
tail -15 $OUT/r2f_host_tests.log
for k in default gather epl0; do
  case $k in default) E="";; gather) E="SC_KERNEL=gather";; epl0) E="SC_EPL=0";; esac
  env $E timeout 600 python bench.py --config 3 --compact --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2f_cfg3c_$k.json 2>&1
  echo "cfg3 compact $k: $(python -c "import json;d=json.loads(open('$OUT/r2f_cfg3c_$k.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
for m in "" "SC_HEAD_CLUSTER=2" "SC_HEAD_CLUSTER=2 SC_HEAD_PAIR_T2=1"; do
  env $m timeout 600 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2f_head.json 2>&1
  echo "head cfg2 [$m]: $(python -c "import json;d=json.loads(open('$OUT/r2f_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
timeout 900 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/r2f_bench_head_cfg3.json 2> $OUT/r2f_bench_head_cfg3.err; tail -c 1800 $OUT/r2f_bench_head_cfg3.json; tail -3 $OUT/r2f_bench_head_cfg3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_r2f_cfg3c -f python bench.py --config 3 --compact --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r2f_cfg3c.ncu-rep --page raw --csv > $OUT/raw_r2f_cfg3c.csv 2>/dev/null
ncu -i $OUT/prof_r2f_cfg3c.ncu-rep --page details --csv > $OUT/details_r2f_cfg3c.csv 2>/dev/null
rm -f $OUT/prof_r2f_cfg3c.ncu-rep
