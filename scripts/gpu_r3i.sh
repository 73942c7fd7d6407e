#!/bin/bash
set -u
OUT=gpurun_out/r3i
mkdir -p $OUT
python scripts/att_vs_T.py c3_nuq3 > $OUT/vsT_c3.txt 2>&1
python scripts/att_vs_T.py c4 > $OUT/vsT_c4.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -rf > $OUT/pytest_parity.txt 2>&1
tail -3 $OUT/pytest_parity.txt
cat $OUT/vsT_c3.txt $OUT/vsT_c4.txt
