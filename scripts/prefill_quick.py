#!/usr/bin/env python
"""Time kvq_prefill_quantize of one C3 layer (131072 tokens) with CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3_nuq3"]
T = 131072
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
K = gen.gen_layer_torch(0, 0, T, w.D, dev, "K")
V = gen.gen_layer_torch(1, 0, T, w.D, dev, "V")
for rep in range(2):
    c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm, capacity_tokens=T,
                     key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"], key_hi=cal["key_hi"], device=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c.prefill(K, V)
    e1.record()
    torch.cuda.synchronize()
    print(f"prefill {T} tokens: {e0.elapsed_time(e1):.2f} ms = {e0.elapsed_time(e1) * 1e6 / T:.1f} ns/token-layer")
    del c
