#!/bin/bash
# round-2 final evidence, session 3 (dense-gradient drain, slot path, lane-per-row all-apps): full GPU suite, smoke, the driver's bench line, the
# reference arm, every NEXT bench line, the N = 2 path on one GPU, ncu launch list + full
# captures of the hot kernels (summaries written on the box).
OUT=gpurun_out
TAG=${TAG:-r4z}
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/${TAG}_pytest_gpu.log 2>&1; echo all_rc=$?; tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $OUT/${TAG}_smoke.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo bench_rc=$?; tail -1 $OUT/${TAG}_bench.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err; tail -1 $OUT/${TAG}_bench_ref.json | cut -c1-200
timeout 600 python bench.py --dtype bf16 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_bf16.json 2>/dev/null
timeout 900 python bench.py --config 3 --compact --steps 50 --warmup 5 --no-cpu-baseline > $OUT/${TAG}_bench_cfg3_compact.json 2>/dev/null
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_bench_cfg3_dense.json 2>/dev/null
timeout 600 python bench.py --config 4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_cfg4.json 2>/dev/null
timeout 600 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_cfg5.json 2>/dev/null
timeout 300 python bench.py --config 2 --order app_choice --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_appchoice.json 2>/dev/null
timeout 300 python bench.py --config 2 --order multi_select --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_multiselect.json 2>/dev/null
timeout 600 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_head.json 2>/dev/null
timeout 900 python bench.py --mode head --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_head_cfg3.json 2>/dev/null
timeout 300 python bench.py --mode ranges --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_ranges.json 2>/dev/null
timeout 300 python bench.py --mode sample --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_sample.json 2>/dev/null
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_allapps.json 2>/dev/null
timeout 300 python bench.py --grad dense --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_dense_f32.json 2>/dev/null
timeout 300 python bench.py --grad dense --dtype bf16 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_dense_bf16.json 2>/dev/null
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --dtype bf16 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_allapps_bf16.json 2>/dev/null
SC_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_bench_n2share.json 2> $OUT/${TAG}_bench_n2share.err
for f in bf16 cfg3_compact cfg3_dense cfg4 cfg5 appchoice multiselect head head_cfg3 ranges sample allapps allapps_bf16 dense_f32 dense_bf16 n2share; do
  echo "$f: $(tail -1 $OUT/${TAG}_bench_$f.json | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('roofline',{});print('%.4g'%d['value'], d.get('unit'), 'ms/step', round(d.get('ms_per_step',0),4), 'frac', round(r.get('frac',0),3), r.get('kernel_ms'))" 2>&1 | tail -1)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_cfg2_f32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_${TAG}_f32 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hist" -s 3 -c 1 -o $OUT/prof_${TAG}_hist -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_cfg3_compact.csv python bench.py --config 3 --compact --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_${TAG}_cfg3c -f python bench.py --config 3 --compact --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_${TAG}_f32.ncu-rep $OUT/${TAG}_launches_cfg2_f32.csv $OUT/ncu_eval_cfg2_f32.json $OUT/${TAG}_eval_cfg2_f32.txt 1048576 eval_kernel > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_${TAG}_hist.ncu-rep $OUT/${TAG}_launches_cfg2_f32.csv $OUT/ncu_hist_cfg2.json $OUT/${TAG}_hist_cfg2.txt 1048576 hist > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_${TAG}_cfg3c.ncu-rep $OUT/${TAG}_launches_cfg3_compact.csv $OUT/ncu_eval_cfg3_compact_f32.json $OUT/${TAG}_eval_cfg3_compact_f32.txt 524288 eval_kernel > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_allapps.csv python bench.py --mode all_apps --config 4 --rows 262144 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"all_apps" -s 1 -c 1 -o $OUT/prof_${TAG}_allapps -f python bench.py --mode all_apps --config 4 --rows 262144 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_${TAG}_allapps.ncu-rep $OUT/${TAG}_launches_allapps.csv $OUT/ncu_allapps_rows_cfg4.json $OUT/${TAG}_allapps_rows_cfg4.txt 262144 all_apps > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_kernels.py > $OUT/${TAG}_sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 $OUT/${TAG}_sanitizer_$tool.log
done
rm -f $OUT/prof_${TAG}_*.ncu-rep
ls $OUT | grep $TAG
