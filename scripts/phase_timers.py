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
ctas = c.info()["splits"] * (w.H_q // c.info()["heads_per_cta"])
print(f"{wname} T={T} attend {e0.elapsed_time(e1) / 5 * 1e3:.1f} us, info {c.info()}")
per = lambda i: round(tm[i] / tiles, 1)
print(f"cycles per tile  K group: tma_wait {per(1)} empty_wait {per(2)} work {per(3)}   "
      f"SV group: full_wait {per(4)} softmax {per(9)} PV {per(10)}")
print(f"prologue cycles per CTA: {tm[0] / (5 * ctas):.0f}")
# one more launch alone for the wall-clock spread across CTAs
c.attend(q, T, o)
torch.cuda.synchronize()
import ctypes
buf = (ctypes.c_uint64 * 4096)()
kvq._lib.kvq_debug_trace(c._h, buf, 4096)
tm = c.phase_timers()
first_start = (~tm[6]) & 0xFFFFFFFFFFFFFFFF
print(f"last launch: first CTA start -> last CTA loop end {(tm[7] - first_start) / 1e3:.1f} us; "
      f"longest CTA start->loop end {tm[8] / 1e3:.1f} us")
# per-tile event trace of CTA 0 (last launch)
if True:
    raw = np.array(buf, dtype=np.uint64).astype(np.int64)
    tr = raw[:3200].reshape(100, 32)
    t0 = tr[0, 0]
    print("tile: K warp starts | K warp ends | SV full softmax pv   (cycles since K start[0])")
    for i in range(0, 10):
        r = tr[i] - t0
        print(i, "K start", r[0:8].tolist(), "end", r[8:16].tolist(), "SV", r[16:19].tolist(), "issue(entry,empty,expect,copies,sync)", r[19:24].tolist(), "SV warps 0/4/7 pre-bar", r[24:27].tolist())
    print("per K warp work / wait per tile (last launch):", [round(int(raw[4000 + k]) / (tm[5] or 1)) for k in range(8)],
          [round(int(raw[4010 + k]) / (tm[5] or 1)) for k in range(8)])
