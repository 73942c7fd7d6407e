"""offline calibration on the GPU (kvq_calibrate_layer) against the oracle's
calibrate_layer (readings R27, R28).

Key thresholds and the Lloyd iteration counts are compared exactly.  The codebooks are fp64
k-means centroids rounded once to fp32 / fp16; the two sides sum the same terms in different
orders (~1e-16 relative), so a stored entry may differ by one unit in the last place when a
centroid sits on a rounding boundary -- the bar is 1 ulp.  Ties in the Values' two-sided split
are exercised with coarse-grained data and per-element Fisher weights (a wrong tie rule moves
weight between points and changes the centroids well beyond 1 ulp)."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import TOL_ATTEND, make_cache, rel_err_per_head

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


def _compare(got, ref):
    for key in ("key_lo", "key_hi"):
        np.testing.assert_array_equal(got[key].view(np.uint32), ref[key].view(np.uint32), key)
    assert tuple(got["iters"]) == tuple(ref["iters"])
    for key in ("cbK", "cbV", "cbK_dec", "cbV_dec"):
        np.testing.assert_array_max_ulp(got[key], ref[key], maxulp=1)
        assert np.all(np.diff(got[key]) > 0), key


def _fisher(seed, N, D):
    rng = np.random.default_rng(seed)
    return (rng.exponential(1.0, (N, D)) * rng.exponential(1.0, (1, D))).astype(np.float32)


@pytest.mark.parametrize("N,D,bits,ppm,fisher,qnorm,fp16,max_iter,tol", [
    (200, 128, 3, 10_000, False, False, True, 100, 1e-6),
    (333, 256, 2, 10_000, True, True, True, 100, 1e-6),
    (257, 128, 4, 20_000, True, False, False, 30, 0.0),
    (1000, 512, 3, 10_000, True, True, False, 60, 1e-7),
    (64, 384, 4, 0, False, True, True, 100, 1e-6),
    (2048, 1024, 3, 10_000, True, False, True, 40, 1e-6),
])
def test_calibrate_matches_oracle(kvq, N, D, bits, ppm, fisher, qnorm, fp16, max_iter, tol):
    K = gen.gen_keys(17, 0, N, D, stream=gen.STREAM_CAL_K)
    V = gen.gen_values(17, 0, N, D, stream=gen.STREAM_CAL_V)
    FK = _fisher(1, N, D) if fisher else None
    FV = _fisher(2, N, D) if fisher else None
    ref = O.calibrate_layer(K, V, bits, ppm, FK=FK, FV=FV, max_iter=max_iter, tol=tol, qnorm=qnorm,
                            fp16_codebooks=fp16)
    Kd, Vd = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    FKd = torch.from_numpy(FK).cuda() if fisher else None
    FVd = torch.from_numpy(FV).cuda() if fisher else None
    got = kvq.calibrate_layer(Kd, Vd, bits, ppm, FKd, FVd, max_iter=max_iter, tol=tol, qnorm=qnorm,
                              fp16_codebooks=fp16)
    _compare(got, ref)
    # host inputs give the same result, and the call is deterministic
    again = kvq.calibrate_layer(K, V, bits, ppm, FK, FV, max_iter=max_iter, tol=tol, qnorm=qnorm,
                                fp16_codebooks=fp16)
    for key in ("cbK", "cbV", "cbK_dec", "cbV_dec", "key_lo", "key_hi"):
        np.testing.assert_array_equal(again[key].view(np.uint32), got[key].view(np.uint32))


@pytest.mark.parametrize("ppm", [10_000, 30_000, 200_000])
def test_calibrate_value_ties(kvq, ppm):
    # Values on a coarse grid: many exact ties at the split; per-element weights decide the result
    rng = np.random.default_rng(ppm)
    N, D = 40, 256
    V = (np.round(rng.standard_normal((N, D)) * 4) / 4).astype(np.float16)
    V[::3, :] = np.float16(0.5)                          # some tokens all equal at the top
    V[1::3, :7] = np.float16(3.0)                        # ties among the largest
    K = rng.standard_normal((N, D)).astype(np.float16)
    FV = rng.exponential(1.0, (N, D)).astype(np.float32) ** 3
    ref = O.calibrate_layer(K, V, 3, ppm, FV=FV, max_iter=50, tol=0.0, fp16_codebooks=False)
    got = kvq.calibrate_layer(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda(), 3, ppm,
                              None, torch.from_numpy(FV).cuda(), max_iter=50, tol=0.0, fp16_codebooks=False)
    _compare(got, ref)


def test_calibrate_errors(kvq):
    K = np.zeros((10, 128), np.float16)
    with pytest.raises(kvq.KVQError):
        kvq.calibrate_layer(K, K, 5, 10_000)
    with pytest.raises(kvq.KVQError):
        kvq.calibrate_layer(K, K, 3, 10_000, max_iter=0)
    with pytest.raises(kvq.KVQError):
        kvq.calibrate_layer(K[:1], K[:1], 3, 400_000)     # too many Key outliers for 1 token
    with pytest.raises(kvq.KVQError):
        kvq.calibrate_layer(np.zeros((10, 100), np.float16), np.zeros((10, 100), np.float16), 3, 10_000)


def test_calibrated_cache_end_to_end(kvq):
    """GPU calibration -> kvq_cache_create -> prefill -> attend, against the oracle run on the
    same calibration result (the product path consumes what f3 produces)."""
    H, bits, ppm, T = 8, 3, 10_000, 777
    D = H * 128
    Kc = gen.gen_keys(5, 0, 4096, D, stream=gen.STREAM_CAL_K)
    Vc = gen.gen_values(5, 0, 4096, D, stream=gen.STREAM_CAL_V)
    cal = kvq.calibrate_layer(torch.from_numpy(Kc).cuda(), torch.from_numpy(Vc).cuda(), bits, ppm, qnorm=True)
    K, V = gen.gen_keys(5, 0, T, D), gen.gen_values(5, 0, T, D)
    q = gen.gen_queries(5, 0, H, H, 128)[0]
    c = make_cache(kvq, cal, H, H, bits, ppm, T)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    o = torch.zeros(H, 128, dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T - 1, o)
    cache = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
    ref = O.attend(cache, q, T - 1, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                   cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
    assert rel_err_per_head(o.cpu().numpy(), ref).max() <= TOL_ATTEND
