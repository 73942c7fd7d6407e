#!/bin/bash
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1
grep -E "passed|failed" $OUT/pytest_gpu.txt | tail -3; grep -E "^FAILED" $OUT/pytest_gpu.txt | head -30
grep -E "^E +assert|^E +AssertionError" $OUT/pytest_gpu.txt | head -40
for T in 65536 131072; do timeout 300 python scripts/prefill_bench.py $T; done > $OUT/prefill.txt 2>&1; cat $OUT/prefill.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -c 1500 $OUT/bench.json
