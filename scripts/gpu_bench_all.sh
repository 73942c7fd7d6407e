#!/bin/bash
# bench lines for every BASELINE config (driver default first), clocks recorded by bench.py
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
timeout 1500 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
tail -c 2500 $OUT/bench_default.json; tail -2 $OUT/bench_default.err
B="python bench.py --no-cpu-baseline --no-compare --steps 10 --warmup 3"
timeout 900 $B --workload c2 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 900 $B --workload c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 $B --workload c3_nuq4 > $OUT/bench_c3_nuq4.json 2> $OUT/bench_c3_nuq4.err
timeout 1500 python bench.py --no-cpu-baseline --no-compare --steps 3 --warmup 3 --workload c5 > $OUT/bench_c5_1gpu.json 2> $OUT/bench_c5_1gpu.err
for f in c2 c4 c3_nuq4 c5_1gpu; do python -c "
import json,sys
try:
  d=json.loads(open('$OUT/bench_$f.json').read().splitlines()[-1])
  print('$f', d['config']['workload'], 'step_ms', round(d['ms_per_step'],3), 'attend_us', round(d['attend_us_per_layer'],1), 'frac', round(d['roofline']['frac'],4), d['config'].get('layer_rule',''))
except Exception as e: print('$f failed', e); print(open('$OUT/bench_$f.err').read()[-800:])
"; done
