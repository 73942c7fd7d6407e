#!/bin/bash
# end-of-session check: smoke, the whole GPU suite, the default bench line
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
tail -1 $OUT/smoke.txt; tail -2 $OUT/pytest_gpu.txt
python -c "
import json
d = json.loads(open('$OUT/bench_default.json').read().strip().splitlines()[-1])
print('value', d['value'], 'attend', d['attend_us_per_layer'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'launches', d.get('gpu_launches'))
"
