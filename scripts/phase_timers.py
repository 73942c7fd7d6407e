#!/usr/bin/env python
"""Per-phase cycle breakdown of att_kernel (diagnostics; run with KVQ_PHASE_TIMERS=1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "c3_nuq3"
w = CONFIGS[wname]
T = int(sys.argv[2]) if len(sys.argv) > 2 else w.T
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm,
                 capacity_tokens=T + 8, key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"],
                 key_hi=cal["key_hi"], device=0)
for a in range(0, T, 65536):
    b = min(T, a + 65536)
    c.prefill(gen.gen_layer_torch(a, 0, b - a, w.D, dev, "K"), gen.gen_layer_torch(a + 1, 0, b - a, w.D, dev, "V"))
c.sync()
q = torch.randn((w.H_q, 128), device=dev).half() * 0.5
o = torch.zeros((w.H_q, 128), device=dev)
for _ in range(3):
    c.attend(q, T, o)
c.sync()
c.phase_timers()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    c.attend(q, T, o)
e1.record()
torch.cuda.synchronize()
tm = c.phase_timers()
tiles = tm[5]
names = ["prologue", "tma_wait", "K_phase", "softmax", "V_phase"]
ctas = info_splits = c.info()["splits"] * (w.H_q // c.info()["heads_per_cta"])
print(f"{wname} T={T} attend {e0.elapsed_time(e1) / 5 * 1e3:.1f} us, info {c.info()}")
print("compute cycles per tile per CTA:", {n: round(tm[i] / tiles, 1) for i, n in enumerate(names)},
      "total", round(sum(tm[1:5]) / tiles, 1))
print(f"prologue cycles per CTA: {tm[0] / (5 * ctas):.0f}  loop cycles per CTA: {sum(tm[1:5]) / (5 * ctas):.0f}")
# one more launch alone for the wall-clock spread across CTAs
c.attend(q, T, o)
torch.cuda.synchronize()
tm = c.phase_timers()
first_start = (~tm[6]) & 0xFFFFFFFFFFFFFFFF
print(f"last launch: first CTA start -> last CTA loop end {(tm[7] - first_start) / 1e3:.1f} us; "
      f"longest CTA start->loop end {tm[8] / 1e3:.1f} us")
