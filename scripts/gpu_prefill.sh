#!/bin/bash
# prefill kernel: parity (codes bit-exact) + timing + ncu capture
set -u
OUT=gpurun_out/${TAG:-pf}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf -k "prefill or append or adversarial or concentrated or host or empty or capacity or full_size or million or large_gqa" > $OUT/pytest.txt 2>&1
tail -25 $OUT/pytest.txt
for T in 4096 65536 131072; do timeout 300 python scripts/prefill_bench.py $T; done > $OUT/prefill.txt 2>&1
cat $OUT/prefill.txt
timeout 300 python scripts/append_bench.py > $OUT/append.txt 2>&1; cat $OUT/append.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 1 -c 1 \
   -o $OUT/prefill python scripts/prefill_bench.py 65536 > $OUT/ncu.txt 2>&1
tail -3 $OUT/ncu.txt
