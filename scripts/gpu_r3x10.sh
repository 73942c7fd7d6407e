#!/bin/bash
# prefill A/B: head vs Key outlier flags gathered 4 pairs at a time (new)
set -u
OUT=gpurun_out/r3x10
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
for v in head new head new; do
  cp build_ab/libkvq_$v.so $L
  echo "$v $(timeout 300 python scripts/prefill_bench.py 131072 2>&1 | tail -1)" >> $OUT/ab.txt
  echo "$v nuq4 $(timeout 300 python scripts/prefill_bench.py 131072 c3_nuq4 2>&1 | tail -1)" >> $OUT/ab.txt
done
cp build_ab/libkvq_new.so $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $OUT/pytest.txt 2>&1
echo "pytest $(tail -1 $OUT/pytest.txt)" >> $OUT/ab.txt
cat $OUT/ab.txt
