#!/bin/bash
# ncu --set full of one att_kernel launch (c3_nuq3, 128K) + per-line summary.  usage: <tag>
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_kernel -s 3 -c 1 \
   -o $OUT/att_full env KVQ_PHASE_TIMERS=1 python scripts/phase_timers.py c3_nuq3 131072 > $OUT/ncu_full.txt 2>&1
tail -3 $OUT/ncu_full.txt
