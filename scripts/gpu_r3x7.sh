#!/bin/bash
# prefill A/B: head vs phase order A, B, publish, C (reord) vs + look-back back-off (both)
set -u
OUT=gpurun_out/r3x7
mkdir -p $OUT
L=paper_2401_18079_b200/libkvq.so
for v in head reord both head reord both; do
  cp build_ab/libkvq_$v.so $L
  echo "$v $(timeout 300 python scripts/prefill_bench.py 131072 2>&1 | tail -1)" >> $OUT/ab.txt
done
for v in head both; do
  cp build_ab/libkvq_$v.so $L
  echo "$v nuq4 $(timeout 300 python scripts/prefill_bench.py 131072 c3_nuq4 2>&1 | tail -1)" >> $OUT/ab.txt
done
cp build_ab/libkvq_both.so $L
KVQ_PHASE_TIMERS=1 timeout 300 python scripts/prefill_phases.py > $OUT/phases.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_online_thresholds.py tests/test_gpu_paged.py -q -x > $OUT/pytest.txt 2>&1
echo "pytest $(tail -1 $OUT/pytest.txt)" >> $OUT/ab.txt
cat $OUT/ab.txt $OUT/phases.txt
