"""GPU parity: CUDA path (through the C ABI) vs the CPU oracle, same seeded inputs.

Bars (north_star):
  * packed codes, outlier indices / values, CSC pointers, per-token (s, z): bit-exact
    (the integer decisions are taken in fp64 on both sides, reading R8);
  * attention output: per query head ||o_gpu - o_ref||_inf / ||o_ref||_inf <= 2e-3, median
    over heads <= 5e-4 (north_star's bar for fp16 products, reading R24, gpu_common).
"""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import (TOL_ATTEND, TOL_ATTEND_MEDIAN, assert_cache_equal, make_cache, tol_attend,
                         merged_partial_to_natural, rel_err_per_head, setup_layer)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = TOL_ATTEND


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


def oracle_cache(cal, K, V, ppm):
    return O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)


def oracle_attend(cal, cache, q, pos, H_q, H_kv, pos_base=0):
    return O.attend(cache, q, pos, H_q=H_q, H_kv=H_kv, d=128, key_lo=cal["key_lo"],
                    key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"],
                    pos_base=pos_base, nthreads=0)


# -------------------------------------------------------------- quantization (T1) --
@pytest.mark.parametrize("H,bits,ppm,T", [(1, 4, 10_000, 77), (2, 3, 10_000, 100),
                                          (2, 2, 10_000, 65), (8, 3, 10_000, 96),
                                          (4, 4, 1_000, 33), (1, 3, 0, 40),
                                          (40, 3, 10_000, 70), (5, 2, 10_000, 45)])
def test_prefill_quantization_bit_exact(kvq, H, bits, ppm, T):
    cal, K, V = setup_layer(1, 0, H, H, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T + 5)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    c.sync()
    assert_cache_equal(c.export(), ref)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_append_then_prefill_mixed(kvq, bits):
    H, ppm, T = 2, 10_000, 70
    cal, K, V = setup_layer(2, 1, H, H, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T)
    Kt, Vt = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    for n in range(5):
        c.append(Kt[n], Vt[n])
    c.prefill(Kt[5:50], Vt[5:50])
    for n in range(50, T):
        c.append(Kt[n], Vt[n])
    c.sync()
    assert c.num_tokens == T
    assert_cache_equal(c.export(), ref)
    assert_cache_equal(c.export(31, 66), ref, 31, 66)


@pytest.mark.parametrize("fill", ["mixed", "prefill"])
def test_adversarial_quantization_inputs(kvq, fill):
    """ties, -0/+0, all-equal tokens, values on midpoints and on thresholds (the prefill
    kernel's exact-selection fallback and its ENC thresholds at midpoints)."""
    H, bits, ppm = 1, 3, 20_000
    D = 128
    cb = np.array([-1.0, -0.5, -0.25, 0.0, 0.25, 0.5, 0.75, 1.0], np.float32)
    lo = np.full(D, -2.0, np.float32)
    hi = np.full(D, 2.0, np.float32)
    cal = dict(cbK=cb, cbV=cb, cbK_dec=cb, cbV_dec=cb, key_lo=lo, key_hi=hi)
    rows_k, rows_v = [], []
    rng = np.random.default_rng(5)
    rows_k.append(np.zeros(D)); rows_v.append(np.zeros(D))                       # all zero
    z = np.zeros(D); z[::2] = -0.0; rows_k.append(z); rows_v.append(z.copy())    # -0 / +0
    rows_k.append(np.full(D, 2.0)); rows_v.append(np.full(D, 3.5))               # == hi, all equal
    mids = np.repeat([-0.75, -0.375, -0.125, 0.125, 0.375, 0.625, 0.875], 19)[:D] * 2.0
    rows_k.append(mids); rows_v.append(np.concatenate([mids[:-2], [7.0, -7.0]]))  # midpoints
    t = rng.choice([-1.0, 0.0, 1.0, 2.0], D); rows_k.append(t); rows_v.append(t)  # heavy ties
    rows_k.append(np.linspace(-3, 3, D)); rows_v.append(np.linspace(-3, 3, D)[::-1].copy())
    K = np.stack(rows_k).astype(np.float16)
    V = np.stack(rows_v).astype(np.float16)
    K[1, ::2] = np.float16(-0.0)
    V[1, ::2] = np.float16(-0.0)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=16)
    Kt, Vt = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    if fill == "prefill":
        c.prefill(Kt, Vt)
    else:
        c.prefill(Kt[:3], Vt[:3])
        for n in range(3, K.shape[0]):
            c.append(Kt[n], Vt[n])
    c.sync()
    assert_cache_equal(c.export(), ref)


def test_host_buffers_are_staged(kvq):
    H, bits, ppm, T = 2, 3, 10_000, 40
    cal, K, V = setup_layer(3, 0, H, H, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T)
    c.prefill(K[:30], V[:30])                      # numpy (pageable host)
    for n in range(30, T):
        c.append(np.ascontiguousarray(K[n]), np.ascontiguousarray(V[n]))
    c.sync()
    assert_cache_equal(c.export(), ref)
    q = gen.gen_queries(3, 0, H, H, 128)[0]
    o = np.zeros((H, 128), np.float32)
    c.attend(q, T - 1, o)
    assert rel_err_per_head(o, oracle_attend(cal, ref, q, T - 1, H, H)).max() < TOL


def test_pinned_host_output_is_stream_ordered(kvq):
    """Page-locked host q / o: the D2H copy stays on the call's stream (kvq.h), so the output
    is valid after a stream synchronize, and equals the device-buffer result."""
    H, bits, ppm, T = 8, 3, 10_000, 300
    cal, K, V = setup_layer(5, 0, H, H, bits, ppm, T)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    q = gen.gen_queries(5, 0, H, H, 128)[0]
    od = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T - 1, od)
    qh = torch.from_numpy(q).pin_memory()
    oh = torch.full((H, 128), -1.0, dtype=torch.float32).pin_memory()
    c.attend(qh, T - 1, oh)
    torch.cuda.synchronize()
    assert torch.equal(oh, od.cpu())


# ----------------------------------------------------------------- attention (T2) --
@pytest.mark.parametrize("H_q,H_kv,bits,T", [(1, 1, 4, 4096), (8, 8, 3, 1000), (2, 2, 4, 333),
                                             (8, 8, 2, 517), (8, 2, 3, 300), (4, 1, 3, 129),
                                             (16, 16, 3, 700), (32, 8, 3, 257),
                                             (8, 4, 3, 301), (16, 8, 2, 400), (32, 16, 3, 96),
                                             (40, 40, 3, 130), (32, 8, 2, 333),
                                             (8, 8, 4, 1000), (32, 32, 4, 300),
                                             # G = 8 (LLaMA-2-70B 64/8): two 4-head CTAs per KV head
                                             (16, 2, 3, 300), (64, 8, 3, 257), (16, 2, 2, 200),
                                             # 4-bit GQA (Mistral-7B nuq4): the tensor-core GQA kernel
                                             (8, 2, 4, 300), (32, 8, 4, 257), (16, 2, 4, 200), (8, 4, 4, 150),
                                             # 40 KV heads of a GQA layer: 40 head groups (> 32: the
                                             # second half of the prefill's per-group scans)
                                             (80, 40, 3, 100), (80, 40, 2, 70)])
def test_attend_matches_oracle(kvq, H_q, H_kv, bits, T):
    ppm = 10_000
    cal, K, V = setup_layer(4, 0, H_q, H_kv, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 64)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    qs = gen.gen_queries(4, 0, H_q, H_kv, 128, n=2)
    for pos, q in zip((T - 1, T + 1000), qs):
        o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), pos, o)
        torch.cuda.synchronize()
        err = rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, pos, H_q, H_kv))
        assert err.max() < tol_attend(H_q, H_kv, bits), err
        assert np.median(err) < TOL_ATTEND_MEDIAN, err


@pytest.mark.parametrize("H_q,H_kv,bits,T", [(8, 8, 3, 1000), (4, 1, 3, 129), (2, 2, 4, 333),
                                             (8, 8, 2, 517)])
def test_attend_fp32_codebook(kvq, H_q, H_kv, bits, T):
    """Decode codebooks that are not fp16 values take the residual pass (R23)."""
    ppm = 10_000
    cal, K, V = setup_layer(14, 0, H_q, H_kv, bits, ppm, T, fp16_codebooks=False)
    assert np.any(cal["cbV_dec"].astype(np.float16).astype(np.float32) != cal["cbV_dec"])
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 64)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    q = gen.gen_queries(14, 0, H_q, H_kv, 128)[0]
    o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    err = rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, T, H_q, H_kv))
    assert err.max() < TOL, err


@pytest.mark.parametrize("splits", [1, 2, 3, 7, 40])
def test_attend_independent_of_split_count(kvq, splits):
    H, bits, ppm, T = 8, 3, 10_000, 1234
    cal, K, V = setup_layer(5, 0, H, H, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    c.set_splits(splits)
    q = gen.gen_queries(5, 0, H, H, 128)[0]
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    assert rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, T, H, H)).max() < TOL


@pytest.mark.parametrize("H_q,H_kv,bits,base", [(2, 2, 3, 9_999_000), (8, 8, 3, 9_990_017),
                                                (32, 8, 3, 9_990_000), (8, 4, 3, 9_999_500),
                                                (8, 8, 2, 8_750_000), (32, 8, 2, 8_750_000),
                                                (8, 8, 4, 9_990_001), (16, 2, 3, 9_990_003),
                                                (8, 2, 4, 8_750_000)])
def test_long_positions_exact_angles(kvq, H_q, H_kv, bits, base):
    """pos_base near 10M (C5 shards start at 8.75M for P = 8): RoPE angles must be reduced
    exactly (reading R12) in every attend kernel -- the two-halves kernel (H = 2), the MHA
    warp-autonomous kernel (H = 8; its per-CTA fp64 anchors and the per-warp fp64 rotation
    recurrence over tiles), the GQA kernel (32/8) and G = 2."""
    ppm, T = 10_000, 600
    cal, K, V = setup_layer(6, 0, H_q, H_kv, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T, pos_base=base)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    for k, pos in enumerate((base + T - 1, base + T + 123_457)):
        q = gen.gen_queries(6 + k, 0, H_q, H_kv, 128)[0]
        o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), pos, o)
        torch.cuda.synchronize()
        err = rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, pos, H_q, H_kv, pos_base=base))
        assert err.max() < TOL, err


def test_sharded_partials_merge_to_unsharded(kvq):
    """Sequence sharding on one GPU: P shards with pos_base, merged."""
    H, bits, ppm, T = 8, 3, 10_000, 999
    cal, K, V = setup_layer(7, 0, H, H, bits, ppm, T)
    ref = oracle_cache(cal, K, V, ppm)
    q = gen.gen_queries(7, 0, H, H, 128)[0]
    qt = torch.from_numpy(q).cuda()
    cuts = [0, 250, 600, 601, 999]
    parts = torch.zeros((len(cuts) - 1, H, 130), dtype=torch.float32, device="cuda")
    caches = []
    for r, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        c = make_cache(kvq, cal, H, H, bits, ppm, capacity=b - a, pos_base=a)
        c.prefill(torch.from_numpy(K[a:b]).cuda(), torch.from_numpy(V[a:b]).cuda())
        c.attend_partial(qt, T, parts[r])
        caches.append(c)
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    kvq.merge_partials(parts, o)
    torch.cuda.synchronize()
    exp = oracle_attend(cal, ref, q, T, H, H)
    assert rel_err_per_head(o.cpu().numpy(), exp).max() < TOL
    # each shard's partial against the oracle's partial on the same shard
    for r, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        sub = oracle_cache(cal, K[a:b], V[a:b], ppm)
        pref = O.attend_partial(sub, q, T, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"],
                                key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"],
                                cbV_dec=cal["cbV_dec"], pos_base=a)
        pg = merged_partial_to_natural(parts[r].cpu().numpy())
        np.testing.assert_allclose(pg[:, -2], pref[:, -2], rtol=1e-3, atol=1e-3)
        og = pg[:, :128] / pg[:, -1:]
        orr = pref[:, :128] / pref[:, -1:]
        assert rel_err_per_head(og, orr).max() < TOL


def test_empty_cache_and_capacity_errors(kvq):
    H, bits, ppm = 1, 3, 10_000
    cal, K, V = setup_layer(8, 0, H, H, bits, ppm, 40)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=32)
    q = torch.zeros((H, 128), dtype=torch.float16, device="cuda")
    o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
    with pytest.raises(kvq.KVQError) as e:
        c.attend(q, 0, o)
    assert e.value.status == kvq.KVQ_EEMPTY
    p = torch.zeros((H, 130), dtype=torch.float32, device="cuda")
    c.attend_partial(q, 0, p)
    assert float(p[0, 129]) == 0.0 and float(p[0, 128]) == float("-inf")
    Kt, Vt = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    c.prefill(Kt[:32], Vt[:32])
    with pytest.raises(kvq.KVQError) as e:
        c.append(Kt[32], Vt[32])
    assert e.value.status == kvq.KVQ_ECAPACITY
    assert c.num_tokens == 32
    c.reset()
    c.prefill(Kt[:7], Vt[:7])
    c.sync()
    assert_cache_equal(c.export(), oracle_cache(cal, K[:7], V[:7], ppm))


def test_key_outlier_capacity_is_sticky(kvq):
    H, bits, ppm, T = 1, 3, 10_000, 64
    cal, K, V = setup_layer(9, 0, H, H, bits, ppm, T)
    cal = dict(cal)
    cal["key_lo"] = np.full(128, -0.01, np.float32)      # nearly everything is an outlier
    cal["key_hi"] = np.full(128, 0.01, np.float32)
    c = make_cache(kvq, cal, H, H, bits, ppm, capacity=T, k_outlier_capacity=100)
    c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    with pytest.raises(kvq.KVQError) as e:
        c.sync()
    assert e.value.status == kvq.KVQ_ECAPACITY


@pytest.mark.parametrize("H_q,H_kv", [(8, 8), (32, 8)])
@pytest.mark.parametrize("fill", ["prefill", "append"])
def test_attend_concentrated_outliers(kvq, H_q, H_kv, fill):
    """Outliers concentrated in one attend bucket group: tile 0 overflows its (tile, group)
    buckets (Key and Value items then come from the CSC / CSR arrays), tile 1 holds more
    items than the attend kernel keeps in registers (the in-bucket slow path), tile 2 is
    ordinary.  Codes bit-exact and attention within the tolerance, MHA and GQA kernels."""
    bits, ppm, T = 3, 10_000, 96
    cal, K, V = setup_layer(21, 0, H_q, H_kv, bits, ppm, T)
    K = K.astype(np.float32)
    V = V.astype(np.float32)
    gqa = H_q != H_kv
    hi = cal["key_hi"].astype(np.float32)
    kch = np.arange(1, 20, 2)                      # 10 Key channels of head 0
    K[0:32, kch] = hi[kch] + 2.0                   # tile 0: > bucket capacity
    if not gqa:
        K[32:64, kch[:4]] = hi[kch[:4]] + 2.0      # tile 1: > 128 items, <= capacity
    kv = -(-ppm * H_kv * 128 // 1_000_000)         # Value outliers per token
    vch = np.arange(0, 2 * kv, 2)                  # kv channels of head 0
    sgn = np.where(np.arange(kv) < (kv + 1) // 2, 1.0, -1.0)
    V[0:32, vch] = 200.0 * sgn                     # tile 0: every outlier in group 0
    n1 = 5 if gqa else 6
    V[32:64, vch[:n1]] = 200.0 * np.where(np.arange(n1) % 2 == 0, 1.0, -1.0)
    K = K.astype(np.float16)
    V = V.astype(np.float16)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 64)
    if fill == "prefill":
        c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    else:
        for n in range(T):
            c.append(np.ascontiguousarray(K[n]), np.ascontiguousarray(V[n]))
    c.sync()
    assert_cache_equal(c.export(), ref)
    q = gen.gen_queries(22, 0, H_q, H_kv, 128)[0]
    o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
    c.attend(torch.from_numpy(q).cuda(), T, o)
    torch.cuda.synchronize()
    err = rel_err_per_head(o.cpu().numpy(), oracle_attend(cal, ref, q, T, H_q, H_kv))
    assert err.max() < TOL, err


# --------------------------------------------------- degenerate / extreme inputs (T2) --
def _extreme_layer(seed, H_q, H_kv, bits, ppm, T, kind):
    cal, K, V = setup_layer(seed, 0, H_q, H_kv, bits, ppm, T)
    K = K.astype(np.float32)
    V = V.astype(np.float32)
    D = H_kv * 128
    rng = np.random.default_rng(seed)
    if kind == "flat_values":
        # tokens whose Value vector is constant: kept range lo == hi, s_n = 0, every code 0
        # (reading R7); with ppm = 0 there are no Value outliers at all
        for n in rng.choice(T, size=T // 3, replace=False):
            V[n, :] = np.float32(rng.normal())
        V[5, :] = 0.0
    elif kind == "huge_value_outliers":
        for n in range(0, T, 3):
            ch = rng.choice(D, size=3, replace=False)
            V[n, ch] = np.array([65504.0, -65504.0, 60000.0])[: len(ch)]
    elif kind == "huge_key_outliers":
        # fp16 Key outliers near +-65504 in many tokens; the score terms they produce exceed
        # 2^15 log2 units (the attend kernels' fixed-point Key-outlier sums must not wrap)
        for n in range(0, T, 4):
            ch = rng.choice(D, size=4, replace=False)
            K[n, ch] = np.array([65504.0, -65504.0, 65000.0, -60000.0])
    return cal, K.astype(np.float16), V.astype(np.float16)


@pytest.mark.parametrize("H_q,H_kv,bits", [(8, 8, 3), (32, 8, 3), (2, 2, 4), (8, 8, 2), (8, 8, 4),
                                           (16, 2, 3), (8, 2, 4)])
@pytest.mark.parametrize("kind,ppm", [("flat_values", 0), ("flat_values", 10_000),
                                      ("huge_value_outliers", 10_000),
                                      ("huge_key_outliers", 10_000)])
def test_attend_extreme_inputs(kvq, H_q, H_kv, bits, kind, ppm):
    """Attention (not only codes) on the method's degenerate and extreme cases: s_n = 0
    tokens, ppm = 0, fp16 Key and Value outliers at +-65504.

    The flat-value construction (a third of the tokens carry a constant random Value vector,
    so |o| is an average of many O(1) constants and small against the inputs) is the hardest
    case for the fp16 products' error budget; the CPU emulation of that
    arithmetic (scripts/prec_emul.py) reproduces the GPU's error on these inputs."""
    T = 161
    cal, K, V = _extreme_layer(31, H_q, H_kv, bits, ppm, T, kind)
    ref = oracle_cache(cal, K, V, ppm)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 8)
    c.prefill(torch.from_numpy(K[:100]).cuda(), torch.from_numpy(V[:100]).cuda())
    for n in range(100, T):
        c.append(torch.from_numpy(K[n]).cuda(), torch.from_numpy(V[n]).cuda())
    c.sync()
    assert_cache_equal(c.export(), ref)
    for k, pos in enumerate((T - 1, T + 77)):
        q = gen.gen_queries(32 + k, 0, H_q, H_kv, 128)[0]
        o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), pos, o)
        torch.cuda.synchronize()
        exp = oracle_attend(cal, ref, q, pos, H_q, H_kv)
        assert np.all(np.isfinite(o.cpu().numpy()))
        err = rel_err_per_head(o.cpu().numpy(), exp)
        assert err.max() < tol_attend(H_q, H_kv, bits), err


@pytest.mark.parametrize("H_q,H_kv,bits", [(8, 8, 3), (32, 8, 3), (8, 8, 2), (2, 2, 4), (8, 8, 4)])
def test_append_then_attend_sees_new_token_pdl(kvq, H_q, H_kv, bits):
    """Decode order with programmatic dependent launch (KVQ_FLAG_DECODE_PDL): each attend is
    enqueued right after the append of the token it must see, with no host sync, across the
    tile boundaries T = 64 and 96 (T = 0 and 31 mod 32).  The appended token is made the
    dominant score (a Key outlier aligned with q at the same position, where q~.k~ = q.k),
    so an attend that missed it would be off by O(1)."""
    ppm, T0, T1 = 10_000, 62, 98
    cal, K, V = setup_layer(41, 0, H_q, H_kv, bits, ppm, T1)
    G = H_q // H_kv
    qs = gen.gen_queries(42, 0, H_q, H_kv, 128, n=T1 - T0)
    K = K.astype(np.float32)
    for n in range(T0, T1):
        q = qs[n - T0].astype(np.float32)
        for h in range(H_kv):
            qh = q[h * G:(h + 1) * G].sum(axis=0)
            c0 = int(np.argmax(np.abs(qh)))
            K[n, h * 128 + c0] = 3000.0 * np.sign(qh[c0])
    K = K.astype(np.float16)
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T1 + 8, decode_pdl=True)
    Kt, Vt = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    c.prefill(Kt[:T0], Vt[:T0])
    qt = torch.from_numpy(qs).cuda()
    outs = torch.zeros((T1 - T0, H_q, 128), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for n in range(T0, T1):
        c.append(Kt[n], Vt[n])
        c.attend(qt[n - T0], n, outs[n - T0])
    torch.cuda.synchronize()
    for n in range(T0, T1):
        pref = O.prefill(K[:n + 1], V[:n + 1], cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
        exp = oracle_attend(cal, pref, qs[n - T0], n, H_q, H_kv)
        err = rel_err_per_head(outs[n - T0].cpu().numpy(), exp)
        assert err.max() < TOL, (n, err)
