#!/bin/bash
set -u
OUT=gpurun_out/r3t
mkdir -p $OUT
python scripts/att_vs_T.py c4 > $OUT/vsT_c4.txt 2>&1
tail -3 $OUT/vsT_c4.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "attend_matches_oracle" > $OUT/pytest.txt 2>&1
tail -2 $OUT/pytest.txt
