#!/bin/bash
# Round-2 final evidence (session 3): smoke, the whole GPU suite, the default bench line (C3 +
# compare arms + CPU baseline + e2e), the other BASELINE configs, the ncu launch list of a C3
# bench and full captures of the attend (MHA, GQA), prefill and append kernels.
set -u
OUT=gpurun_out/${TAG:-r2c}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> $OUT/host.txt
python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 1200 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 python bench.py --workload c3_nuq4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_nuq4.json 2> $OUT/bench_c3_nuq4.err
timeout 1500 python bench.py --workload c5 --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c5_1gpu.json 2> $OUT/bench_c5_1gpu.err
KS="regex:att_|prefill_kernel|append_kernel|merge_kernel|f16_"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KS" --csv \
   --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --layers 4 \
   --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_wa_kernel -s 6 -c 1 \
   -o $OUT/att_wa python scripts/att_ab.py c3_nuq3 > $OUT/ncu_wa.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:att_wag_kernel -s 6 -c 1 \
   -o $OUT/att_wag python scripts/att_ab.py c4 262144 > $OUT/ncu_wag.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 2 -c 1 \
   -o $OUT/prefill python scripts/prefill_quick.py > $OUT/ncu_prefill.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:append_kernel -s 20 -c 1 \
   -o $OUT/append python scripts/append_bench.py > $OUT/ncu_append.txt 2>&1
python - <<P
import json
for n in ("default", "c2", "c4", "c3_nuq4", "c5_1gpu"):
    try:
        d = json.loads(open("$OUT/bench_%s.json" % n).read().strip().splitlines()[-1])
        print(n, d["value"], d.get("attend_us_per_layer"), d["roofline"]["frac"], d.get("clocks"))
    except Exception as e:
        print(n, "ERR", e)
P
