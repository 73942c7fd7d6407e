#!/usr/bin/env python
"""Time (and, under ncu, profile) single-token kvq_append on the C3 layer shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

w = CONFIGS["c3_nuq3"]
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
n = 64
c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm, capacity_tokens=4096,
                 key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"], key_hi=cal["key_hi"], device=0)
K = gen.gen_layer_torch(0, 0, n, w.D, dev, "K")
V = gen.gen_layer_torch(1, 0, n, w.D, dev, "V")
for i in range(8):
    c.append(K[i], V[i])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(8, n):
    c.append(K[i], V[i])
e1.record()
torch.cuda.synchronize()
print(f"append: {e0.elapsed_time(e1) / (n - 8) * 1e3:.1f} us per token (D={w.D}, b={w.bits})")
