#!/usr/bin/env python
"""Attention error of the C4 shape (GQA 32/8, 3-bit, 1% outliers) against the fp64 oracle at
a long context: per-head max relative error of the bench launch configuration.
usage: diag_gqa.py [T] [workload]   (KVQ_ATT_LEGACY=1 selects the two-halves kernel)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from kvq_synth import CONFIGS, calib, gen  # noqa: E402
from paper_2401_18079_b200 import kvq  # noqa: E402
from tests.gpu_common import make_cache, rel_err_per_head  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
w = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c4"]
D, H, Hk = w.D, w.H_q, w.H_kv
cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, D, stream=gen.STREAM_CAL_K),
                            gen.gen_values(0, 0, 2048, D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
Kt = gen.gen_layer_torch(7, 0, T, D, "cpu", "K")
Vt = gen.gen_layer_torch(8, 0, T, D, "cpu", "V")
c = make_cache(kvq, cal, H, Hk, w.bits, w.ppm, capacity=T + 32)
for a in range(0, T, 262144):
    b = min(T, a + 262144)
    c.prefill(Kt[a:b].cuda(), Vt[a:b].cuda())
ref = O.prefill(Kt.numpy(), Vt.numpy(), cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm, kcap=64 * T)
q = gen.gen_queries(9, 0, H, Hk, 128)[0]
o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
c.attend(torch.from_numpy(q).cuda(), T, o)
torch.cuda.synchronize()
e = O.attend(ref, q, T, H_q=H, H_kv=Hk, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
             cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
r = rel_err_per_head(o.cpu().numpy().astype(np.float64), e)
tag = "legacy" if os.environ.get("KVQ_ATT_LEGACY") else "default"
print(f"{w.name} T={T} {tag} kernel={c.info()['attend_kernel']}: max rel {r.max():.2e} median {np.median(r):.2e}; "
      f"worst heads {np.argsort(r)[-4:][::-1].tolist()} {np.sort(r)[-4:][::-1].round(6).tolist()}; "
      f"max|o| of those {np.abs(e).max(-1)[np.argsort(r)[-4:][::-1]].round(4).tolist()}")
