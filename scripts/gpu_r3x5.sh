#!/bin/bash
# prefill A/B: head vs L2 prefetch of the next head slices (pf) vs + next V row in phase A (pfa)
set -u
OUT=gpurun_out/r3x5
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
for v in head pf pfa head pf pfa; do
  cp build_ab/libkvq_$v.so $L
  echo "$v $(timeout 300 python scripts/prefill_bench.py 131072 2>&1 | tail -1)" >> $OUT/ab.txt
done
for v in head pf pfa; do
  cp build_ab/libkvq_$v.so $L
  echo "$v nuq4 $(timeout 300 python scripts/prefill_bench.py 131072 c3_nuq4 2>&1 | tail -1)" >> $OUT/ab.txt
done
cat $OUT/ab.txt
