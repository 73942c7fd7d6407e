#!/bin/bash
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
B="python bench.py --no-cpu-baseline --no-e2e --no-compare"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:att_wa_kernel -s 3 -c 1 \
   -o $OUT/att_wa $B --steps 1 --warmup 3 --layers 2 > $OUT/ncu_wa.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:att_wag_kernel -s 3 -c 1 \
   -o $OUT/att_wag $B --workload c4 --steps 1 --warmup 3 --layers 2 > $OUT/ncu_wag.txt 2>&1
ls $OUT
