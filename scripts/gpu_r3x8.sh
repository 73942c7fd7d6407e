#!/bin/bash
set -u
OUT=gpurun_out/r3x8
mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 1 -c 1 \
   -o $OUT/prefill python scripts/prefill_bench.py 65536 > $OUT/ncu.txt 2>&1
tail -2 $OUT/ncu.txt
