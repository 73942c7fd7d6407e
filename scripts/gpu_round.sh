#!/bin/bash
# One gpurun call: tests, smoke, bench, launch list, ncu capture of the attend kernel.
# usage: scripts/gpu_round.sh <tag> [bench args...]
set -u
TAG=${1:-r}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> $OUT/host.txt
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
tail -5 $OUT/pytest_gpu.txt
timeout 1200 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
