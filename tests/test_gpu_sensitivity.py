"""mixed-precision sensitivity on the GPU (kvq_layer_sensitivity,
kvq_fisher_accumulate, kvq_assign_bits) against the oracle (eq:opt2 P:1336-1339 over the
oracle's own prefill + dequantize).  Omega is an fp64 sum whose order differs between the two
sides (atomics on the GPU), so the bar is 1e-9 relative; the assignment is compared exactly."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import make_cache, setup_layer

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


def _fisher(seed, T, D):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((T, D)) ** 2 * rng.exponential(1.0, (1, D))).astype(np.float32)


@pytest.mark.parametrize("H_kv,bits,T,prefix,fisher", [
    (1, 2, 1, 0, False), (4, 3, 77, 0, True), (8, 4, 300, 0, True), (2, 3, 100, 45, True),
    (32, 3, 2048, 0, True), (8, 2, 513, 31, False)])
def test_layer_sensitivity_matches_oracle(kvq, H_kv, bits, T, prefix, fisher):
    ppm = 10_000
    cal, K, V = setup_layer(61 + bits, 0, H_kv, H_kv, bits, ppm, prefix + T)
    D = H_kv * 128
    Ks, Vs = K[prefix:], V[prefix:]
    FK = _fisher(5, T, D) if fisher else None
    FV = _fisher(6, T, D) if fisher else None
    ok, ov = O.layer_omega(Ks, Vs, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm,
                           FK=FK, FV=FV, cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
    c = make_cache(kvq, cal, H_kv, H_kv, bits, ppm, prefix + T + 8)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    Kd, Vd = torch.from_numpy(Ks).cuda(), torch.from_numpy(Vs).cuda()
    FKd = torch.from_numpy(FK).cuda() if fisher else None
    FVd = torch.from_numpy(FV).cuda() if fisher else None
    om = kvq.layer_sensitivity(c, Kd, Vd, FKd, FVd, t0=prefix)             # host output
    assert om[0] == pytest.approx(ok, rel=REL) and om[1] == pytest.approx(ov, rel=REL)
    # host inputs, device output
    od = torch.zeros(2, dtype=torch.float64, device="cuda")
    kvq.layer_sensitivity(c, Ks, Vs, FK, FV, t0=prefix, omega=od)
    torch.cuda.synchronize()
    np.testing.assert_allclose(od.cpu().numpy(), [ok, ov], rtol=REL)


def test_layer_sensitivity_errors(kvq):
    cal, K, V = setup_layer(3, 0, 1, 1, 3, 10_000, 40)
    c = make_cache(kvq, cal, 1, 1, 3, 10_000, 64)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    with pytest.raises(kvq.KVQError):
        kvq.layer_sensitivity(c, K, V, t0=1)          # [1, 41) is not cached
    om = kvq.layer_sensitivity(c, K[:0], V[:0], t0=40)
    assert om[0] == 0.0 and om[1] == 0.0


def test_fisher_accumulate(kvq):
    rng = np.random.default_rng(8)
    gs = rng.standard_normal((3, 1000)).astype(np.float32)
    F = torch.zeros(1000, dtype=torch.float32, device="cuda")
    for g in gs:
        kvq.fisher_accumulate(F, torch.from_numpy(g).cuda())
    torch.cuda.synchronize()
    np.testing.assert_allclose(F.cpu().numpy(), O.fisher_diag(list(gs.astype(np.float64))), rtol=1e-6)


def test_assign_bits_matches_oracle(kvq):
    np.testing.assert_array_equal(kvq.assign_bits([5, 1, 3], 1, 4, 2), [4, 2, 4])
    np.testing.assert_array_equal(kvq.assign_bits([2, 2, 2], 2, 3, 2), [2, 2, 3])
    with pytest.raises(kvq.KVQError):
        kvq.assign_bits([1, 2], 3, 4, 2)
    with pytest.raises(kvq.KVQError):
        kvq.assign_bits([1, float("nan")], 1, 4, 2)


def test_mixed_precision_end_to_end(kvq):
    """Four layers with different statistics: Omega at the lower precision (3 bits) with Fisher
    weights on the GPU, one-shot assignment, then the per-layer caches at the assigned widths
    attend within the R24 bar (each against the oracle at its own width)."""
    from .gpu_common import TOL_ATTEND, rel_err_per_head
    ppm, T, H = 10_000, 600, 4
    oms_gpu, oms_ref, setups = [], [], []
    for layer in range(4):
        cal, K, V = setup_layer(90, layer, H, H, 3, ppm, T)
        V = (V.astype(np.float32) * (1.0 + layer)).astype(np.float16)      # distinct sensitivities
        FK, FV = _fisher(20 + layer, T, H * 128), _fisher(30 + layer, T, H * 128)
        ref = O.layer_omega(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm, FK=FK, FV=FV,
                            cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
        c = make_cache(kvq, cal, H, H, 3, ppm, T)
        c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
        om = kvq.layer_sensitivity(c, K, V, FK, FV)
        np.testing.assert_allclose(om, ref, rtol=REL)
        oms_gpu.append(float(om.sum()))
        oms_ref.append(sum(ref))
        setups.append((layer, K, V))
    bits = kvq.assign_bits(oms_gpu, 2, 4, 3)
    demoted = O.assign_mixed_precision(oms_ref, 2)
    np.testing.assert_array_equal(np.flatnonzero(bits == 3), demoted)
    q = gen.gen_queries(90, 0, H, H, 128)[0]
    for layer, K, V in setups:
        b = int(bits[layer])
        cal, _, _ = setup_layer(90, layer, H, H, b, ppm, 1)
        c = make_cache(kvq, cal, H, H, b, ppm, T)
        c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
        o = torch.zeros(H, 128, dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), T - 1, o)
        o = o.cpu().numpy()
        cache = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
        ref = O.attend(cache, q, T - 1, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                       cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
        assert rel_err_per_head(o, ref).max() <= TOL_ATTEND
