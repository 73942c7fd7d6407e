#!/bin/bash
set -u
OUT=gpurun_out/r3n
mkdir -p $OUT
python scripts/att_vs_T.py c4 > $OUT/vsT_c4_wgt.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "8-2 or 4-1 or 8-4 or 16-8 or 32-16 or 32-8 or G or gqa" > $OUT/pytest.txt 2>&1
tail -2 $OUT/pytest.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_wgt_kernel -s 6 -c 1 \
   -o $OUT/wgt python scripts/att_ab.py c4 262144 > $OUT/ncu_wgt.txt 2>&1
cat $OUT/vsT_c4_wgt.txt
