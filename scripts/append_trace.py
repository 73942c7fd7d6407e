#!/usr/bin/env python
"""Single-token append on the C3 layer shape: (a) GPU time per append from CUDA-graph replays of
32 appends (no host overhead), (b) with KVQ_PHASE_TIMERS=1, the phase clocks of append_kernel
(globaltimer ns after: staging, Values warp, Keys warps, sync, CSC slot, records, V codes)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_nuq3"
w = CONFIGS[name]
dev = torch.device("cuda", 0)
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, w.D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, w.D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
n = 96
c = kvq.KVQCache(n_q_heads=w.H_q, n_kv_heads=w.H_kv, bits=w.bits, outlier_ppm=w.ppm, capacity_tokens=4096,
                 key_cb=cal["cbK"], val_cb=cal["cbV"], key_lo=cal["key_lo"], key_hi=cal["key_hi"], device=0,
                 trust_device_ptrs=True)
K = gen.gen_layer_torch(0, 0, n, w.D, dev, "K")
V = gen.gen_layer_torch(1, 0, n, w.D, dev, "V")
for i in range(8):
    c.append(K[i], V[i])
torch.cuda.synchronize()
if os.environ.get("KVQ_PHASE_TIMERS"):
    lib = kvq.lib()
    lib.kvq_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(16, np.uint64)
    tmp = np.zeros(16, np.uint64)
    rows = []
    for i in range(8, 72):
        c.phase_timers()          # resets the trace region
        c.append(K[i], V[i])
        torch.cuda.synchronize()
        lib.kvq_debug_trace(c.handle, buf.ctypes.data, 16)
        r_ = buf.astype(np.int64) - int(buf[0])
        r_[15] = int(buf[15])
        rows.append(r_)
    r = np.median(np.array(rows[8:]), axis=0)
    names = ["start", "staged", "v:finish(w0)", "keys_warps", "sync1", "csc_slot", "records", "vcodes_end",
             "v:selected", "-", "-", "-", "-", "-", "-", "-"]
    print("phase ends (ns from kernel start, median of 56):")
    for nm, v in zip(names, r):
        if nm != "-":
            print(f"  {nm:12s} {v:8.0f}")
else:
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            for i in range(8, 40):
                c.append(K[i], V[i], s)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"append ({name}): {e0.elapsed_time(e1) / (20 * 32) * 1e3:.2f} us per token, graph-replayed")
