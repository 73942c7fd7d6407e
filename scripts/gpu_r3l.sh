#!/bin/bash
set -u
OUT=gpurun_out/r3l
mkdir -p $OUT
python scripts/att_vs_T.py c4 > $OUT/vsT_c4_wgt.txt 2>&1
KVQ_WGT_OFF=1 python scripts/att_vs_T.py c4 > $OUT/vsT_c4_wag.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf > $OUT/pytest.txt 2>&1
tail -4 $OUT/pytest.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -c 1 \
   -o $OUT/prefill python scripts/prefill_quick.py > $OUT/ncu_prefill.txt 2>&1
cat $OUT/vsT_c4_wgt.txt $OUT/vsT_c4_wag.txt
