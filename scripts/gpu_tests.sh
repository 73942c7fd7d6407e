#!/bin/bash
# One gpurun call: smoke + the GPU test suite (no -x: report every failure).
# usage: scripts/gpu_tests.sh <tag> [pytest args...]
set -u
TAG=${1:-t}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 "$@" > $OUT/pytest_gpu.txt 2>&1
tail -40 $OUT/pytest_gpu.txt
cat $OUT/smoke.txt | tail -3
