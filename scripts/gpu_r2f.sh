#!/bin/bash
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1
grep -E "passed|failed" $OUT/pytest_gpu.txt | tail -3; grep -E "^FAILED" $OUT/pytest_gpu.txt | head -30
grep -E "^E +assert|^E +AssertionError|Error" $OUT/pytest_gpu.txt | head -20
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 4000 $OUT/bench.json; tail -3 $OUT/bench.err
