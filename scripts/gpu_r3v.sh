#!/bin/bash
set -u
OUT=gpurun_out/r3v
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -rf > $OUT/pytest.txt 2>&1
tail -4 $OUT/pytest.txt
timeout 1200 python bench.py --workload l70b --steps 5 --warmup 3 --no-cpu-baseline --no-compare > $OUT/bench_l70b.json 2> $OUT/bench_l70b.err
python -c "
import json
d = json.loads(open('$OUT/bench_l70b.json').read().strip().splitlines()[-1])
print('l70b', d['value'], d.get('attend_us_per_layer'), d['roofline']['frac'])
"
python scripts/diag_attend_err.py > $OUT/diag.txt 2>&1; tail -6 $OUT/diag.txt
