#!/bin/bash
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded_2proc.py -q -rf -x > $OUT/pytest.txt 2>&1
grep -E "passed|failed" $OUT/pytest.txt | tail -2; grep -E "^FAILED|^E +(assert|Assert)" $OUT/pytest.txt | head
timeout 300 python scripts/append_bench.py; KVQ_OLD_APPEND=1 timeout 300 python scripts/append_bench.py
B="python bench.py --no-cpu-baseline --no-e2e --no-compare --steps 10 --warmup 3"
timeout 600 $B > $OUT/c3.json 2>$OUT/c3.err; python -c "import json;d=json.loads(open('$OUT/c3.json').read().splitlines()[-1]);print('C3', d['ms_per_step'], d['attend_us_per_layer'], d['roofline']['frac'], d['append_us_per_layer'])"
