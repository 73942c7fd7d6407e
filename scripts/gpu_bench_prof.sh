#!/bin/bash
# bench + ncu launch list + ncu full capture of att_kernel.  usage: <tag> [bench args]
set -u
TAG=${1:-r}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
tail -c 4000 $OUT/bench.json; tail -3 $OUT/bench.err
KS="regex:att_|qz_kernel|scan_counts|merge_kernel|sort_buckets"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KS" --csv \
   --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --layers 4 \
   --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.txt 2>&1
tail -2 $OUT/ncu_launch_bench.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 3 -c 1 \
   -o $OUT/att_full python bench.py --steps 1 --warmup 1 --layers 2 --no-cpu-baseline --no-e2e \
   > $OUT/ncu_full.txt 2>&1
tail -3 $OUT/ncu_full.txt
