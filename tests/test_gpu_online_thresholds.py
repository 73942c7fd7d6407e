"""online per-channel Key thresholds ("Online for K") on the
GPU (kvq_key_thresholds_online) against the oracle's order statistics: bit-exact, including
ties, -0 / +0, n = 0 and blocks smaller than a CTA's row slice; then an end-to-end prefill with
the online thresholds (codes bit-exact, attention within the R24 bar)."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import calib, gen

from .gpu_common import TOL_ATTEND, assert_cache_equal, make_cache, rel_err_per_head

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


@pytest.mark.parametrize("T,D,ppm", [(1, 128, 0), (5, 128, 10_000), (777, 256, 10_000), (4096, 4096, 10_000),
                                     (20_000, 1024, 1_000), (3000, 128, 200_000), (64, 192, 0)])
def test_online_thresholds_bit_exact(kvq, T, D, ppm):
    K = gen.gen_keys(71, 0, T, D)
    K[T // 2, : D // 2] = np.float16(-0.0)                 # signed zeros
    if T > 10:
        K[: T // 3, 7] = np.float16(1.5)                   # heavy ties in one channel
    lo_ref, hi_ref = O.key_thresholds_online(K, ppm)
    lo, hi = kvq.key_thresholds_online(torch.from_numpy(K).cuda(), ppm)        # host outputs
    np.testing.assert_array_equal(lo.view(np.uint32), lo_ref.view(np.uint32))
    np.testing.assert_array_equal(hi.view(np.uint32), hi_ref.view(np.uint32))
    lo_d = torch.zeros(D, dtype=torch.float32, device="cuda")
    hi_d = torch.zeros(D, dtype=torch.float32, device="cuda")
    kvq.key_thresholds_online(K, ppm, lo_d, hi_d)                             # host input, device outputs
    torch.cuda.synchronize()
    np.testing.assert_array_equal(lo_d.cpu().numpy().view(np.uint32), lo_ref.view(np.uint32))
    np.testing.assert_array_equal(hi_d.cpu().numpy().view(np.uint32), hi_ref.view(np.uint32))


def test_online_thresholds_errors(kvq):
    K = torch.zeros((1, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(kvq.KVQError) as e:
        kvq.key_thresholds_online(K, 10_000)               # n = 1 outlier of 1 token: nothing kept
    assert e.value.status == kvq.KVQ_EINVAL


@pytest.mark.parametrize("H,bits", [(8, 3), (8, 4)])
def test_prefill_with_online_thresholds(kvq, H, bits):
    """'Online for K': thresholds from the prompt's own Keys, then the usual prefill / attend."""
    ppm, T = 10_000, 900
    D = H * 128
    cal = calib.calibrate_layer(gen.gen_keys(72, 0, 2048, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(72, 0, 2048, D, stream=gen.STREAM_CAL_V), bits, ppm)
    K, V = gen.gen_keys(73, 0, T, D), gen.gen_values(73, 0, T, D)
    lo, hi = kvq.key_thresholds_online(torch.from_numpy(K).cuda(), ppm)
    lo_ref, hi_ref = O.key_thresholds_online(K, ppm)
    np.testing.assert_array_equal(lo, lo_ref)
    cal = dict(cal, key_lo=lo_ref, key_hi=hi_ref)
    ref = O.prefill(K, V, lo_ref, hi_ref, cal["cbK"], cal["cbV"], ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    c.sync()
    assert_cache_equal(c.export(), ref)
    q = gen.gen_queries(74, 0, H, H, 128)[0]
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    exp = O.attend(ref, q, T, H_q=H, H_kv=H, d=128, key_lo=lo_ref, key_hi=hi_ref, cbK_dec=cal["cbK_dec"],
                   cbV_dec=cal["cbV_dec"])
    assert rel_err_per_head(o.cpu().numpy(), exp).max() < TOL_ATTEND
