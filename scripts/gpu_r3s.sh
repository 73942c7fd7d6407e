#!/bin/bash
set -u
OUT=gpurun_out/r3s
mkdir -p $OUT
timeout 1500 python bench.py --workload c4_nuq4 --steps 5 --warmup 3 --no-cpu-baseline --no-compare > $OUT/bench_c4_nuq4.json 2> $OUT/bench_c4_nuq4.err
timeout 1500 python bench.py --workload l70b --steps 5 --warmup 3 --no-cpu-baseline --no-compare > $OUT/bench_l70b.json 2> $OUT/bench_l70b.err
for f in c4_nuq4 l70b; do python -c "
import json
d = json.loads(open('$OUT/bench_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['unit'], d.get('attend_us_per_layer'), d['roofline']['frac'], d['roofline']['kernel'])
"; tail -2 $OUT/bench_$f.err; done
