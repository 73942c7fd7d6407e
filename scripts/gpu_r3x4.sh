#!/bin/bash
set -u
OUT=gpurun_out/r3x4
mkdir -p $OUT
KVQ_PHASE_TIMERS=1 timeout 300 python scripts/prefill_phases.py > $OUT/prefill_phases.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 1 -c 1 \
   -o $OUT/prefill python scripts/prefill_bench.py 65536 > $OUT/ncu.txt 2>&1
cat $OUT/prefill_phases.txt; tail -2 $OUT/ncu.txt
