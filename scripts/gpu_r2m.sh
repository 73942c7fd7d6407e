#!/bin/bash
# full GPU suite + smoke + default bench (f3/f4 arms included)
set -u
OUT=gpurun_out/r2m
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu.txt 2>&1
tail -5 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 600 $OUT/bench.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/r2m/bench.json").read().strip().splitlines()[-1])
for k in ("value", "ms_per_step", "offline_calibration", "sensitivity", "online_key_thresholds", "batched_decode"):
    print(k, json.dumps(d.get(k))[:400])
print("roofline", d["roofline"])
P
