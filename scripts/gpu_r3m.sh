#!/bin/bash
set -u
OUT=gpurun_out/r3m
mkdir -p $OUT
python scripts/diag_attend_err.py > $OUT/diag_wgt.txt 2>&1
KVQ_WGT_OFF=1 python scripts/diag_attend_err.py > $OUT/diag_wag.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_wgt_kernel -s 6 -c 1 \
   -o $OUT/wgt python scripts/att_ab.py c4 262144 > $OUT/ncu_wgt.txt 2>&1
grep " 8 \| 4 \| 16 " $OUT/diag_wgt.txt; echo; grep " 8 \| 4 \| 16 " $OUT/diag_wag.txt
