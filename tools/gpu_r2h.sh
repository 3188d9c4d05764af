#!/bin/bash
# r2h: dense-mapped key fix (parity + cfg3-compact bench), head knob sweep + ncu, NEXT rooflines (all-apps).
OUT=gpurun_out
timeout 900 python -m pytest tests/test_compact_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2h_tests.log 2>&1; echo tests_rc=$?
tail -3 $OUT/r2h_tests.log
for dt in f32 bf16; do
  timeout 600 python bench.py --config 3 --dtype $dt --compact --steps 50 --warmup 5 --no-cpu-baseline > $OUT/r2h_cfg3c_$dt.json 2>&1
  echo "cfg3 compact $dt: $(python -c "import json;d=json.loads(open('$OUT/r2h_cfg3c_$dt.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3), round(d['value']/1e9,3),'G/s', 'e2e', round(d['e2e']['value']/1e6,2), d['e2e'].get('host_mode'))")"
done
for m in "" "SC_HEAD_KBS=1" "SC_HEAD_KBS=4" "SC_HEAD_WSTAGES=5" "SC_HEAD_KBS=1 SC_HEAD_WSTAGES=5" "SC_HEAD_T2=0"; do
  env $m timeout 600 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2h_head.json 2>&1
  echo "head cfg2 [$m]: $(python -c "import json;d=json.loads(open('$OUT/r2h_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
done
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2h_bench_allapps.json 2>&1; tail -c 900 $OUT/r2h_bench_allapps.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 2 -c 1 -o $OUT/prof_r2h_head -f python bench.py --mode head --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2h_launches_head.csv python bench.py --mode head --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_r2h_head.ncu-rep $OUT/r2h_launches_head.csv $OUT/ncu_head_cfg2_d2048.json $OUT/r2h_head_cfg2_d2048.txt 1048576 head_kernel > /dev/null 2>&1
ncu -i $OUT/prof_r2h_head.ncu-rep --page raw --csv > $OUT/raw_r2h_head.csv 2>/dev/null
rm -f $OUT/prof_r2h_head.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"all_apps" -s 1 -c 1 -o $OUT/prof_r2h_allapps -f python bench.py --mode all_apps --config 4 --rows 262144 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2h_launches_allapps.csv python bench.py --mode all_apps --config 4 --rows 262144 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_r2h_allapps.ncu-rep $OUT/r2h_launches_allapps.csv $OUT/ncu_allapps_cfg4.json $OUT/r2h_allapps_cfg4.txt 262144 all_apps > /dev/null 2>&1
rm -f $OUT/prof_r2h_allapps.ncu-rep
ls $OUT | tail -20
