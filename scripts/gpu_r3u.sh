#!/bin/bash
set -u
OUT=gpurun_out/r3u
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
tail -2 $OUT/smoke.txt
timeout 900 python -m pytest tests/test_gpu_batch.py -q -rf > $OUT/pytest_batch.txt 2>&1
tail -3 $OUT/pytest_batch.txt
