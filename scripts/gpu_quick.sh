#!/bin/bash
# quick GPU check: parity tests (fail fast) + one bench line.  usage: <tag> [bench args...]
set -u
TAG=${1:-q}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
tail -15 $OUT/pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline "$@" > $OUT/bench.json 2> $OUT/bench.err
tail -c 1500 $OUT/bench.json; tail -3 $OUT/bench.err
