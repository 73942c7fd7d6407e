#!/bin/bash
# session start: full GPU suite + smoke + default bench at HEAD
set -u
OUT=gpurun_out/r3a
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu.txt 2>&1
tail -5 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 600 $OUT/bench.err
python -c "
import json
d = json.loads(open('gpurun_out/r3a/bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'attend', d.get('attend_us_per_layer'), 'prefill', d.get('prefill'), 'append', d.get('append'))
print('roofline', d['roofline'])
"
