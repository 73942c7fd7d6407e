#!/bin/bash
# prefill 4-bit: 2 vs 3 CTAs/SM (mix = 4-bit at 2, nv3 = all at 3), head for reference
set -u
OUT=gpurun_out/r3x3
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
for v in head mix nv3 mix nv3; do
  cp build_ab/libkvq_$v.so $L
  echo "$v $(timeout 300 python scripts/prefill_bench.py 131072 c3_nuq4 2>&1 | tail -1)" >> $OUT/ab.txt
done
cp build_ab/libkvq_mix.so $L
echo "mix c3_nuq3 $(timeout 300 python scripts/prefill_bench.py 131072 2>&1 | tail -1)" >> $OUT/ab.txt
cat $OUT/ab.txt
