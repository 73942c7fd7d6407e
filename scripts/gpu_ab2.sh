#!/bin/bash
# A/B + parity + append timing, everything into gpurun_out/<tag>/out.txt
set -u
TAG=${1:-ab}; W=${2:-c3_nuq3}; T=${3:-0}
OUT=gpurun_out/$TAG
mkdir -p $OUT
{
bash scripts/gpu_ab.sh $TAG $W $T
python scripts/append_bench.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -2
} > $OUT/out.txt 2>&1
cat $OUT/out.txt
