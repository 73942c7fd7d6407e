#!/bin/bash
set -u
OUT=gpurun_out/r3q
mkdir -p $OUT
KVQ_PHASE_TIMERS=1 timeout 300 python scripts/prefill_phases.py > $OUT/prefill_phases.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_wgt_kernel -s 3 -c 1 \
   -o $OUT/wgt_c4_1m python bench.py --workload c4 --steps 1 --warmup 1 --layers 2 --no-cpu-baseline --no-e2e --no-compare > $OUT/ncu_wgt.txt 2>&1
cat $OUT/prefill_phases.txt | tail -20; tail -2 $OUT/ncu_wgt.txt
