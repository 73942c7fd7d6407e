#!/bin/bash
# A/B of the GQA score mma: tf32 hi + lo (build default) vs fp16 hi + lo (build_ab/libkvq_f16.so)
set -u
OUT=gpurun_out/r3w
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
cp $L build_ab/cur.so
timeout 600 python scripts/att_vs_T.py c4 > $OUT/tf32_c4.txt 2>&1
timeout 600 python scripts/att_vs_T.py l70b > $OUT/tf32_l70b.txt 2>&1
cp build_ab/libkvq_f16.so $L
timeout 600 python scripts/att_vs_T.py c4 > $OUT/f16_c4.txt 2>&1
timeout 600 python scripts/att_vs_T.py l70b > $OUT/f16_l70b.txt 2>&1
cp build_ab/cur.so $L
timeout 300 python scripts/diag_attend_err.py > $OUT/diag.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -rf -k "gqa or GQA or wgt or 8" > $OUT/pytest.txt 2>&1
tail -3 $OUT/pytest.txt
tail -3 $OUT/tf32_c4.txt $OUT/f16_c4.txt $OUT/tf32_l70b.txt $OUT/f16_l70b.txt
grep "kernel 2" $OUT/diag.txt
