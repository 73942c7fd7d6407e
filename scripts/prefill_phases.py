#!/usr/bin/env python
"""Prefill phase shares (KVQ_PHASE_TIMERS=1): CTA clock sums per phase of prefill_kernel
(A Value selection, C Value codes + B Keys, D1, D1b, D2) for one C3 layer of 65536 tokens."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

w = CONFIGS["c3_nuq3"]
T = 65536
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
K = gen.gen_layer_torch(0, 0, T, w.D, dev, "K")
V = gen.gen_layer_torch(1, 0, T, w.D, dev, "V")
c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm, capacity_tokens=T,
                 key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"], key_hi=cal["key_hi"], device=0)
c.phase_timers()
c.prefill(K, V)
c.sync()
lib = kvq.lib()
lib.kvq_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(72, np.uint64)
lib.kvq_debug_trace(c.handle, buf.ctypes.data, 72)
ph = buf[64:70].astype(np.float64)
names = ["init", "A: V select", "B: Keys", "D1 + C: V codes", "D1b", "D2"]
tot = ph.sum()
for n_, v in zip(names, ph):
    print(f"  {n_:22s} {100 * v / tot:5.1f}%   {v / (T / 32) / 1.9e3:8.1f} us per CTA-tile")
