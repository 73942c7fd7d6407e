#!/bin/bash
# prefill A/B: HEAD vs Value mask in warp scratch (2 CTAs/SM) vs same at 3 CTAs/SM
set -u
OUT=gpurun_out/r3x2
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
for v in head nv2 nv3 head nv2 nv3; do
  cp build_ab/libkvq_$v.so $L
  echo "$v $(timeout 300 python scripts/prefill_bench.py 131072 2>&1 | tail -1)" >> $OUT/ab.txt
done
for v in nv2 nv3; do
  cp build_ab/libkvq_$v.so $L
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_online_thresholds.py tests/test_gpu_paged.py -q -x > $OUT/pytest_$v.txt 2>&1
  echo "$v $(tail -1 $OUT/pytest_$v.txt)" >> $OUT/ab.txt
done
cat $OUT/ab.txt
