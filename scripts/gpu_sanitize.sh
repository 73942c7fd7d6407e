#!/bin/bash
# compute-sanitizer memcheck / racecheck / initcheck / synccheck on the tiny T1/T2 cases
set -u
OUT=gpurun_out/${TAG}/sanitizer
mkdir -p $OUT
SEL='test_prefill_quantization_bit_exact[2-3-10000-100] or test_attend_matches_oracle[8-8-3-1000] or test_attend_matches_oracle[32-8-3-257] or test_attend_matches_oracle[2-2-4-333] or test_append_then_attend_sees_new_token_pdl[8-8-3] or test_f16_cache_store_and_attend[8-1000-0]'
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --target-processes all \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16.py -q -k "$SEL" -p no:cacheprovider \
     > $OUT/$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/$tool.txt | tr '\n' ' ')"
done
