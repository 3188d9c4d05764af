#!/bin/bash
for cfg in "SC_HEAD_WSTAGES=4" "SC_HEAD_WSTAGES=5" "SC_HEAD_WSTAGES=6" "SC_HEAD_WSTAGES=7" "SC_HEAD_WSTAGES=5 SC_HEAD_KBS=1" "SC_HEAD_WSTAGES=5 SC_HEAD_KBS=2" "SC_HEAD_WSTAGES=6 SC_HEAD_KBS=2" "SC_HEAD_WSTAGES=4 SC_HEAD_KBS=4"; do
  env SC_HEAD_CLUSTER=1 $cfg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum.per_second,launch__shared_mem_per_block_dynamic --clock-control none -k regex:head_kernel -c 1 python bench.py --mode head --d 2048 --steps 1 --warmup 1 2>/dev/null | grep -E "gpu__time|dram__|shared" | tail -3 | tr '\n' ' '; echo " <- $cfg"
done
for cfg in "SC_HEAD_WSTAGES=5" "SC_HEAD_WSTAGES=3"; do
  env SC_HEAD_CLUSTER=1 $cfg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum.per_second --clock-control none -k regex:head_kernel -c 1 python bench.py --mode head --d 512 --steps 1 --warmup 1 2>/dev/null | grep -E "gpu__time|dram__" | tail -2 | tr '\n' ' '; echo " <- d512 $cfg"
done
