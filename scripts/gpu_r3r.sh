#!/bin/bash
set -u
OUT=gpurun_out/r3r
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf > $OUT/pytest_parity.txt 2>&1
tail -6 $OUT/pytest_parity.txt
python scripts/att_vs_T.py c4 > $OUT/vsT_c4.txt 2>&1
tail -2 $OUT/vsT_c4.txt
