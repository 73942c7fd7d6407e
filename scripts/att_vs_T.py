#!/usr/bin/env python
"""Attend time per launch against context length, CUDA-graph replayed (no host launch cost):
the intercept is the kernel's fixed cost (prologue, merge, tail).  usage: att_vs_T.py [workload]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, EXTRA_CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "c3_nuq3"
w = CONFIGS[wname] if wname in CONFIGS else EXTRA_CONFIGS[wname]
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
torch.manual_seed(0)
q = torch.randn((w.H_q, 128), device=dev).half() * 0.5
for T in (32, 1024, 4096, 16384, 65536, 131072):
    caches = []
    for L in range(4):
        c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm,
                         capacity_tokens=T + 8, key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"],
                         key_hi=cal["key_hi"], device=0)
        for a in range(0, T, 65536):
            b = min(T, a + 65536)
            c.prefill(gen.gen_layer_torch(a + 7 * L, 0, b - a, w.D, dev, "K"),
                      gen.gen_layer_torch(a + 7 * L + 1, 0, b - a, w.D, dev, "V"))
        c.sync()
        caches.append(c)
    o = torch.zeros((4, w.H_q, 128), device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for L, c in enumerate(caches):
            c.attend(q, T, o[L], stream=s.cuda_stream)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for L, c in enumerate(caches):
            c.attend(q, T, o[L], stream=s.cuda_stream)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{wname} T={T}: {e0.elapsed_time(e1) / (n * 4) * 1e3:.1f} us per attend (graph)", flush=True)
    del caches
