#!/bin/bash
# ncu evidence: launch list of a short bench, full captures of the hot kernels
set -u
OUT=gpurun_out/${TAG}
mkdir -p $OUT
B="python bench.py --no-cpu-baseline --no-e2e --no-compare"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:att_|qz_kernel|prefill_kernel|merge_kernel|f16_" --csv \
   --log-file $OUT/launches.csv $B --steps 2 --warmup 3 --layers 4 > $OUT/launch_bench.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:att_wa_kernel -s 3 -c 1 \
   -o $OUT/att_wa $B --steps 1 --warmup 3 --layers 2 > $OUT/ncu_wa.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:att_wag_kernel -s 3 -c 1 \
   -o $OUT/att_wag $B --workload c4 --steps 1 --warmup 3 --layers 2 > $OUT/ncu_wag.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qz_kernel -s 5 -c 1 \
   -o $OUT/append $B --steps 1 --warmup 3 --layers 2 > $OUT/ncu_append.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 1 -c 1 \
   -o $OUT/prefill python scripts/prefill_bench.py 65536 > $OUT/ncu_prefill.txt 2>&1
timeout 300 python scripts/append_bench.py > $OUT/append.txt 2>&1
KVQ_NO_PDL=1 timeout 600 $B --steps 10 --warmup 3 > $OUT/bench_nopdl.json 2>&1
timeout 600 $B --steps 10 --warmup 3 > $OUT/bench_pdl.json 2>&1
tail -c 300 $OUT/bench_nopdl.json; tail -c 300 $OUT/bench_pdl.json; cat $OUT/append.txt
ls $OUT
