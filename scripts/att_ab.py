#!/usr/bin/env python
"""A/B timing of the attend kernels on one layer (KVQ_ATT_LEGACY=1 selects the two-halves
kernel).  usage: att_ab.py [workload] [tokens] [out.npy]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "c3_nuq3"
w = CONFIGS[wname]
T = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else w.T
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
caches = []
for L in range(4):   # 4 layers cycled so no launch reads a layer out of L2
    c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm,
                     capacity_tokens=T + 8, key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"],
                     key_hi=cal["key_hi"], device=0)
    for a in range(0, T, 65536):
        b = min(T, a + 65536)
        c.prefill(gen.gen_layer_torch(a + 7 * L, 0, b - a, w.D, dev, "K"),
                  gen.gen_layer_torch(a + 7 * L + 1, 0, b - a, w.D, dev, "V"))
    c.sync()
    caches.append(c)
torch.manual_seed(0)
q = torch.randn((w.H_q, 128), device=dev).half() * 0.5
o = torch.zeros((4, w.H_q, 128), device=dev)
for _ in range(3):
    for L, c in enumerate(caches):
        c.attend(q, T, o[L])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    for L, c in enumerate(caches):
        c.attend(q, T, o[L])
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / (n * 4) * 1e3
tag = "legacy" if os.environ.get("KVQ_ATT_LEGACY") else "default"
print(f"{wname} T={T} {tag}: attend {us:.1f} us/layer, info {caches[0].info()}")
if len(sys.argv) > 3:
    np.save(sys.argv[3], o.cpu().numpy())
