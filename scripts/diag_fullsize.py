#!/usr/bin/env python
"""Diagnose attention error at the C3 size: per-head partials (m, l, o) GPU vs oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402
from tests.gpu_common import make_cache, merged_partial_to_natural  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
w = CONFIGS["c3_nuq3"]
D, H = w.D, w.H_q
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
Kt = gen.gen_layer_torch(7, 0, T, D, "cpu", "K")
Vt = gen.gen_layer_torch(8, 0, T, D, "cpu", "V")
c = make_cache(kvq, cal, H, H, w.bits, w.ppm, capacity=T + 32)
c.prefill(Kt.cuda(), Vt.cuda())
ref = O.prefill(Kt.numpy(), Vt.numpy(), cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm, kcap=64 * T)
q = gen.gen_queries(9, 0, H, H, 128)[0]
part = torch.zeros((H, 130), dtype=torch.float32, device="cuda")
c.attend_partial(torch.from_numpy(q).cuda(), T, part)
torch.cuda.synchronize()
g = merged_partial_to_natural(part.cpu().numpy())
e = O.attend_partial(ref, q, T, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                     cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"], pos_base=0, nthreads=0)
for h in range(H):
    # compare normalized outputs and log-sum-exp
    og, oe = g[h, :128] / g[h, 129], e[h, :128] / e[h, 129]
    lse_g = g[h, 128] + np.log(g[h, 129])
    lse_e = e[h, 128] + np.log(e[h, 129])
    rel = np.abs(og - oe).max() / np.abs(oe).max()
    print(f"head {h:2d} rel {rel:.2e}  lse gpu {lse_g:.6f} ora {lse_e:.6f} d {lse_g - lse_e:+.2e}  "
          f"max|o| {np.abs(oe).max():.3e}  m {e[h,128]:.3f}  l {e[h,129]:.1f}")
