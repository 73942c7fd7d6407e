#!/bin/bash
# GPU evidence for the bench lines and profiles (TAG env = output dir): smoke, GPU tests, default bench (C3 + oracle CPU
# baseline), C2 / C4 / C5-shard / C3-4bit bench lines, ncu launch list + full captures of the
# MHA and GQA attend kernels.
set -u
OUT=gpurun_out/${TAG:-r1d}
mkdir -p $OUT
bash scripts/gpu_round.sh ${TAG:-r1d} > $OUT/round.txt 2>&1
timeout 600 python bench.py --workload c2 --no-cpu-baseline > $OUT/bench_c2.json 2>$OUT/bench_c2.err
timeout 1200 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2>$OUT/bench_c4.err
timeout 900 python bench.py --workload c5 --tokens 1250000 --layers 4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.json 2>$OUT/bench_c5.err
timeout 900 python bench.py --workload c3_nuq4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_nuq4.json 2>$OUT/bench_c3_nuq4.err
KS="regex:att_|qz_kernel|scan_counts|merge_kernel|sort_buckets"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KS" --csv \
   --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --layers 4 \
   --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 3 -c 1 \
   -o $OUT/att_full python bench.py --steps 1 --warmup 1 --layers 2 --no-cpu-baseline --no-e2e \
   > $OUT/ncu_full.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 3 -c 1 \
   -o $OUT/att_full_c4 python bench.py --workload c4 --steps 1 --warmup 1 --layers 2 --no-cpu-baseline --no-e2e \
   > $OUT/ncu_full_c4.txt 2>&1
tail -3 $OUT/round.txt
