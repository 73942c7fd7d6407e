#!/bin/bash
# ncu --set full of one attend launch (default kernel selection) on C3.  usage: <tag> [workload] [tokens]
set -u
TAG=${1:-nwa}; W=${2:-c3_nuq3}; T=${3:-0}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python scripts/att_ab.py $W $T 2>&1 | tail -1
KVQ_WA_WH=${WH:-2} timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 6 -c 1 \
   -o $OUT/att_full python scripts/att_ab.py $W $T > $OUT/ncu_full.txt 2>&1
tail -3 $OUT/ncu_full.txt
