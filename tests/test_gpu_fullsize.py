"""Parity at the benchmarked size (BASELINE config C3 / bench.py default): one LLaMA-7B layer
(32 heads x 128), 131072 cached tokens, 3-bit NUQ, 1% outliers, the launch configuration
bench.py times (automatic head grouping and split count).  The oracle quantizes the same
seeded input (OpenMP over tokens) and computes attention for every head in fp64; the GPU
codes of sampled tokens are compared bit-exactly and the attention output within the
north_star tolerance.  Slow (~1-2 min): inputs 2 x 1 GiB fp16."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_synth import CONFIGS, calib, gen

from .gpu_common import TOL_ATTEND as TOL, TOL_ATTEND_MEDIAN, assert_cache_equal, make_cache, rel_err_per_head, tol_attend

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as K
    return K


@pytest.mark.parametrize("fp16_codebooks", [True, False])
def test_c3_full_size_layer(kvq, fp16_codebooks):
    """fp16_codebooks=False keeps the fp32 k-means centroids, which exercises the attend
    kernel's residual pass for the V codebook (R23)."""
    w = CONFIGS["c3_nuq3"]
    T, D, H = w.T, w.D, w.H_q
    assert (T, D, H, w.bits) == (131072, 4096, 32, 3)
    cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(0, 0, 2048, D, stream=gen.STREAM_CAL_V), w.bits, w.ppm,
                                fp16_codebooks=fp16_codebooks)
    Kt = gen.gen_layer_torch(7, 0, T, D, "cpu", "K")
    Vt = gen.gen_layer_torch(8, 0, T, D, "cpu", "V")
    K = Kt.numpy()
    V = Vt.numpy()

    c = make_cache(kvq, cal, H, H, w.bits, w.ppm, capacity=T + 32)
    c.prefill(Kt.cuda(), Vt.cuda())
    c.sync()
    ref = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm, kcap=64 * T)

    # every canonical array of sampled token windows (start, middle, ragged tail) bit-exact:
    # codes, Value (s, z), Value outliers, Key CSC pointers / channels / values
    for t0 in (0, 65_531, T - 40):
        assert_cache_equal(c.export(t0, t0 + 40), ref, t0, t0 + 40)
    # the whole Key CSC pointer array and Value (s, z) at full size
    e = c.export(0, T)
    np.testing.assert_array_equal(e["kptr"] - e["kptr"][0], ref.kptr - ref.kptr[0])
    np.testing.assert_array_equal(e["vs"].view(np.uint32), ref.vs.view(np.uint32))
    np.testing.assert_array_equal(e["vz"].view(np.uint32), ref.vz.view(np.uint32))
    np.testing.assert_array_equal(e["kidx"].astype(np.int32), ref.kidx)
    np.testing.assert_array_equal(e["kval"], ref.kval)

    q = gen.gen_queries(9, 0, H, H, 128)[0]
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    exp = O.attend(ref, q, T, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                   cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"], pos_base=0, nthreads=0)
    err = rel_err_per_head(o.cpu().numpy(), exp)
    print("C3 full-size per-head max rel err: max %.3g median %.3g" % (err.max(), np.median(err)))
    assert err.max() < TOL and np.median(err) < TOL_ATTEND_MEDIAN, err


@pytest.mark.parametrize("wname,T", [("c4", 65536), ("c5", 65536)])
def test_large_gqa_and_qnorm_layers(kvq, wname, T):
    """C4 (Mistral GQA 32/8, 3-bit) and C5 (2-bit, Q-Norm decode codebooks) layer shapes at
    65536 tokens, the bench launch configuration; every head against the oracle."""
    w = CONFIGS[wname]
    D, H, Hk = w.D, w.H_q, w.H_kv
    cal = calib.calibrate_layer(gen.gen_keys(1, 0, 2048, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(1, 0, 2048, D, stream=gen.STREAM_CAL_V), w.bits, w.ppm,
                                qnorm=w.qnorm)
    Kt = gen.gen_layer_torch(17, 0, T, D, "cpu", "K", param_seed=1)
    Vt = gen.gen_layer_torch(18, 0, T, D, "cpu", "V", param_seed=1)
    c = make_cache(kvq, cal, H, Hk, w.bits, w.ppm, capacity=T + 32)
    c.prefill(Kt.cuda(), Vt.cuda())
    c.sync()
    ref = O.prefill(Kt.numpy(), Vt.numpy(), cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm,
                    kcap=64 * T)
    assert_cache_equal(c.export(T - 40, T), ref, T - 40, T)
    q = gen.gen_queries(19, 0, H, Hk, 128)[0]
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    exp = O.attend(ref, q, T, H_q=H, H_kv=Hk, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                   cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"], pos_base=0, nthreads=0)
    err = rel_err_per_head(o.cpu().numpy(), exp)
    print("%s T=%d per-head max rel err: max %.3g median %.3g" % (wname, T, err.max(), np.median(err)))
    assert err.max() < tol_attend(H, Hk, w.bits) and np.median(err) < TOL_ATTEND_MEDIAN, err


@pytest.mark.slow
def test_c4_million_tokens(kvq):
    """C4 at its BASELINE size: Mistral-7B GQA 32/8 layer, 1,048,576 cached tokens, 3-bit,
    the GQA kernel in the bench launch configuration; every head against the fp64 oracle."""
    w = CONFIGS["c4"]
    T, D, H, Hk = w.T, w.D, w.H_q, w.H_kv
    assert T == 1 << 20
    cal = calib.calibrate_layer(gen.gen_keys(2, 0, 2048, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(2, 0, 2048, D, stream=gen.STREAM_CAL_V), w.bits, w.ppm)
    Kt = gen.gen_layer_torch(27, 0, T, D, "cpu", "K", param_seed=2)
    Vt = gen.gen_layer_torch(28, 0, T, D, "cpu", "V", param_seed=2)
    c = make_cache(kvq, cal, H, Hk, w.bits, w.ppm, capacity=T + 32)
    c.prefill(Kt.cuda(), Vt.cuda())
    c.sync()
    ref = O.prefill(Kt.numpy(), Vt.numpy(), cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm,
                    kcap=64 * T)
    for t0 in (0, T // 2 + 3, T - 40):
        assert_cache_equal(c.export(t0, t0 + 40), ref, t0, t0 + 40)
    for k in range(2):
        q = gen.gen_queries(29 + k, 0, H, Hk, 128)[0]
        o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), T + 5 * k, o)
        torch.cuda.synchronize()
        exp = O.attend(ref, q, T + 5 * k, H_q=H, H_kv=Hk, d=128, key_lo=cal["key_lo"],
                       key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"],
                       pos_base=0, nthreads=0)
        err = rel_err_per_head(o.cpu().numpy(), exp)
        print("C4 1M per-head max rel err: max %.3g median %.3g" % (err.max(), np.median(err)))
        assert err.max() < tol_attend(H, Hk, w.bits) and np.median(err) < TOL_ATTEND_MEDIAN, err
