#!/bin/bash
# ncu --set full of the MHA (C3) and GQA (C4, 256K tokens) attend kernels at HEAD
set -u
OUT=gpurun_out/r3b
mkdir -p $OUT
timeout 300 python scripts/att_ab.py c3_nuq3 > $OUT/ab_c3.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 6 -c 1 \
   -o $OUT/wa python scripts/att_ab.py c3_nuq3 > $OUT/ncu_wa.txt 2>&1
timeout 300 python scripts/att_ab.py c4 262144 > $OUT/ab_c4.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_ -s 6 -c 1 \
   -o $OUT/wag python scripts/att_ab.py c4 262144 > $OUT/ncu_wag.txt 2>&1
cat $OUT/ab_c3.txt $OUT/ab_c4.txt; tail -2 $OUT/ncu_wa.txt $OUT/ncu_wag.txt
