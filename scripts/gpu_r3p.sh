#!/bin/bash
set -u
OUT=gpurun_out/r3p
mkdir -p $OUT
timeout 1500 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -rf -s -k "c4 or million" > $OUT/pytest_fullsize_c4.txt 2>&1
grep -E "rel err|passed|failed" $OUT/pytest_fullsize_c4.txt | tail -5
python -c "
import json
d = json.loads(open('$OUT/bench_c4.json').read().strip().splitlines()[-1])
print(d['value'], d.get('attend_us_per_layer'), d['roofline'], d.get('clocks'))
"
