"""Per-head attention error of the MHA attend kernel on the parity-test layers (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from kvq_synth import gen  # noqa: E402
from paper_2401_18079_b200 import kvq as K_  # noqa: E402
from tests.gpu_common import make_cache, rel_err_per_head, setup_layer  # noqa: E402
from tests.test_gpu_parity import oracle_attend, oracle_cache  # noqa: E402

for (H, Hk, bits, T) in [(16, 2, 3, 300), (64, 8, 3, 257), (16, 2, 2, 200), (40, 40, 3, 130), (8, 8, 3, 1000), (16, 16, 3, 700), (8, 8, 2, 517), (32, 8, 3, 257), (8, 4, 3, 301), (16, 8, 2, 400), (32, 16, 3, 96), (32, 8, 2, 333)]:
    cal, K, V = setup_layer(4, 0, H, Hk, bits, 10_000, T)
    ref = oracle_cache(cal, K, V, 10_000)
    c = make_cache(K_, cal, H, Hk, bits, 10_000, capacity=T + 64)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    qs = gen.gen_queries(4, 0, H, Hk, 128, n=2)
    for pos, q in zip((T - 1, T + 1000), qs):
        o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), pos, o)
        torch.cuda.synchronize()
        err = rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, pos, H, Hk))
        print(H, Hk, bits, T, pos, "kernel", c.info()["attend_kernel"], "max %.3e median %.3e argmax %d" % (err.max(), np.median(err), err.argmax()))
