#!/usr/bin/env python
"""Time kvq_prefill_quantize (block quantization) on the C3 layer shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3_nuq3"]
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
K = gen.gen_layer_torch(0, 0, T, w.D, dev, "K")
V = gen.gen_layer_torch(1, 0, T, w.D, dev, "V")
c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm, capacity_tokens=4 * T,
                 key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"], key_hi=cal["key_hi"], device=0)
c.prefill(K, V)   # warm
c.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    c.prefill(K, V)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
rd = T * w.D * 2 * 2
print(f"prefill T={T}: {ms:.3f} ms = {ms * 1e6 / T:.1f} ns/token-layer, fp16 K+V read {rd / ms / 1e6:.0f} GB/s")
