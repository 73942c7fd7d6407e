#!/bin/bash
set -u
OUT=gpurun_out/r3o
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf > $OUT/pytest_parity.txt 2>&1
tail -4 $OUT/pytest_parity.txt
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "test_attend_matches_oracle and (32-8-3 or 16-2-3 or 8-4-3)" > $OUT/sanitizer_memcheck_wgt.txt 2>&1
tail -4 $OUT/sanitizer_memcheck_wgt.txt
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "test_attend_matches_oracle and (8-4-3 or 16-2-3)" > $OUT/sanitizer_racecheck_wgt.txt 2>&1
tail -4 $OUT/sanitizer_racecheck_wgt.txt
