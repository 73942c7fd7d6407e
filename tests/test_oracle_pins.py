"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: a value the paper
(or SPEC's hand derivation of it) prints, a closed form, an invariant, a different
formulation (matrix RoPE, exact-rational argmin, dominance property of the outlier
split), or textbook attention on a lossless cache.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from kvq_synth import gen


# ---------------------------------------------------------------------------- RoPE --
def test_rope_golden(golden):
    g = golden("rope.json")
    for c in g["cases"]:
        out = O.rope(np.array(c["x"]), c["pos"])
        np.testing.assert_allclose(out, c["out"], rtol=0, atol=1e-15)


def _paper_matrix_rope(x_adj, pos, base=10000.0):
    """Block-diagonal matrix of P:699-708 acting on ADJACENT pairs (x_{2i-1}, x_{2i})."""
    d = x_adj.shape[0]
    R = np.zeros((d, d))
    for i in range(1, d // 2 + 1):
        th = base ** (-2.0 * (i - 1) / d)
        c, s = np.cos(pos * th), np.sin(pos * th)
        a, b = 2 * (i - 1), 2 * (i - 1) + 1
        R[a, a], R[a, b], R[b, a], R[b, b] = c, -s, s, c
    return R @ x_adj


@pytest.mark.parametrize("d,pos", [(4, 1), (8, 1000), (128, 12345), (128, 9_999_999)])
def test_rope_equals_matrix_form_up_to_pairing(d, pos):
    # element-wise form is "different but equivalent": pairs (i, i+d/2) instead of
    # (2i-1, 2i).  Interleave, apply the paper's matrix, de-interleave.
    x = np.random.default_rng(d + pos).standard_normal(d)
    half = d // 2
    x_adj = np.empty(d)
    x_adj[0::2], x_adj[1::2] = x[:half], x[half:]
    y_adj = _paper_matrix_rope(x_adj, pos)
    expect = np.concatenate([y_adj[0::2], y_adj[1::2]])
    np.testing.assert_allclose(O.rope(x, pos), expect, rtol=0, atol=1e-12)


def test_rope_norm_and_relative_position():
    rng = np.random.default_rng(0)
    q, k = rng.standard_normal(128), rng.standard_normal(128)
    assert abs(np.linalg.norm(O.rope(q, 777)) - np.linalg.norm(q)) < 1e-12
    # Eq. rope1: score depends only on n - m.
    base = O.rope(q, 5) @ O.rope(k, 3)
    for shift in (1, 4096, 10_000_000):
        shifted = O.rope(q, 5 + shift) @ O.rope(k, 3 + shift)
        assert abs(shifted - base) <= 1e-9 * max(1.0, abs(base))


# ----------------------------------------------------------------------------- ENC --
def test_enc_golden(golden):
    g = golden("enc.json")
    for y, code in g["cases"]:
        assert O.enc(y, g["s"], g["z"], g["codebook"]) == code, y


def _argmin_exact(y, s, z, cb):
    """Nearest centroid to (y - z)/s with exact rationals, ties to the lower index."""
    s, z = Fraction(float(s)), Fraction(float(z))
    if s == 0:
        return 0
    yn = (Fraction(float(y)) - z) / s
    best, bd = 0, None
    for j, c in enumerate(cb):
        dist = abs(yn - Fraction(float(c)))
        if bd is None or dist < bd:
            best, bd = j, dist
    return best


def test_enc_matches_exact_rational_argmin():
    rng = np.random.default_rng(1)
    for trial in range(3000):
        nlev = int(rng.choice([4, 8, 16]))
        cb = np.sort(rng.uniform(-1.2, 1.2, nlev)).astype(np.float32)
        cb = np.unique(cb)
        s = np.float32(abs(rng.standard_normal()) * 3 + 1e-3)
        z = np.float32(rng.standard_normal())
        if trial % 3 == 0:
            # aim exactly at a midpoint (ties) when representable
            j = int(rng.integers(0, cb.size - 1))
            y = np.float16(float(z) + float(s) * (float(cb[j]) + float(cb[j + 1])) / 2)
        else:
            y = np.float16(rng.standard_normal() * 3)
        assert O.enc(float(y), float(s), float(z), cb) == _argmin_exact(y, s, z, cb)


def test_enc_on_grid_hits_and_tie_lower():
    cb = np.array([-1.0, -0.25, 0.0, 0.5], np.float32)
    for j, c in enumerate(cb):
        assert O.enc(float(c) * 2 + 1, 2.0, 1.0, cb) == j
    # midpoint of -0.25 and 0 (= -0.125) -> lower index 1
    assert O.enc(-0.125, 1.0, 0.0, cb) == 1
    # s = 0 (degenerate range, reading R7) -> code 0
    assert O.enc(3.0, 0.0, 3.0, cb) == 0


# ---------------------------------------------------------------- outlier split --
def test_outlier_split_golden(golden):
    g = golden("outlier_split.json")
    for c in g["cases"]:
        v = np.array(c["v"], np.float16)
        mask = O.select_outliers(v, c["k"])
        assert sorted(np.nonzero(mask)[0].tolist()) == c["outliers"]
        kept = v[~mask].astype(np.float64)
        assert kept.min() == np.float64(np.float16(c["lo"]))
        assert kept.max() == np.float64(np.float16(c["hi"]))
    for D, ppm, k in g["counts"]:
        assert O.outlier_count(D, ppm) == k


def _dominates_desc(a, b, v):   # a ranks before b in (value desc, index asc)
    return v[a] > v[b] or (v[a] == v[b] and a < b)


def _dominates_asc(a, b, v):
    return v[a] < v[b] or (v[a] == v[b] and a < b)


@pytest.mark.parametrize("D", [2, 3, 5, 8])
def test_outlier_split_dominance_bruteforce(D):
    """Exhaustive tie patterns: the upper set dominates everything outside it; the lower
    set dominates the remainder (ascending); -0 ties with +0."""
    rng = np.random.default_rng(D)
    pool = np.array([-1.0, -0.0, 0.0, 1.0, 2.0], np.float16)
    for _ in range(400):
        v = rng.choice(pool, D)
        vv = v.astype(np.float64)
        for k in range(0, D):
            mask = O.select_outliers(v, k)
            assert mask.sum() == k
            ku, kl = (k + 1) // 2, k // 2
            idx = np.nonzero(mask)[0]
            # recover U as the ku best by desc order among the masked
            upper = [i for i in range(D) if mask[i] and all(
                _dominates_desc(i, j, vv) for j in range(D) if not mask[j])]
            assert len(upper) >= ku
            # there is a choice of U (size ku) dominating all non-U; check via ranks
            rank = sorted(range(D), key=lambda i: (-vv[i], i))
            U = set(rank[:ku])
            rest = [i for i in range(D) if i not in U]
            L = set(sorted(rest, key=lambda i: (vv[i], i))[:kl])
            assert set(idx.tolist()) == U | L


# ------------------------------------------------------------------ quantization --
def test_normalize_worked_example():
    # v=[0,2,4] with lo=0, hi=4 -> s=2, z=2, normalized [-1, 0, 1]
    s, z = O.affine_from_range(0.0, 4.0)
    assert (s, z) == (2.0, 2.0)
    cb = np.array([-1.0, 0.0, 1.0, 1.5], np.float32)
    codes, idx, val = O.quantize_key(np.array([0, 2, 4], np.float16), [0, 0, 0], [4, 4, 4], cb)
    assert codes.tolist() == [0, 1, 2] and idx.size == 0


def test_key_threshold_semantics():
    cb = np.array([-1.0, -0.3, 0.3, 1.0], np.float32)
    lo = np.array([-1.0, -1.0, -1.0, -1.0], np.float32)
    hi = np.array([1.0, 1.0, 1.0, 1.0], np.float32)
    x = np.array([1.0, 1.5, -1.0, -2.0], np.float16)  # == hi kept, > hi out, == lo kept, < lo out
    codes, idx, val = O.quantize_key(x, lo, hi, cb)
    assert idx.tolist() == [1, 3]
    assert val.view(np.float16).tolist() == [1.5, -2.0]
    assert codes.tolist() == [3, 3, 0, 0]   # outlier slots hold ENC(clamp(x)) (reading R5)


def test_value_quant_roundtrip_bounds_and_exact_outliers():
    rng = np.random.default_rng(3)
    cb = np.array([-1.0, -0.6, -0.25, 0.0, 0.2, 0.45, 0.7, 1.0], np.float32)
    gap = np.max(np.diff(cb.astype(np.float64)))
    for _ in range(50):
        v = (rng.standard_normal(256) * 2).astype(np.float16)
        codes, idx, val, s, z = O.quantize_value(v, 10_000, cb)
        assert idx.size == 3
        deq = cb[codes].astype(np.float64) * s + z
        deq[idx] = val.view(np.float16).astype(np.float64)
        err = np.abs(deq - v.astype(np.float64))
        assert np.all(err[idx] == 0)
        kept = np.setdiff1d(np.arange(256), idx)
        assert np.all(err[kept] <= s * gap / 2 * (1 + 1e-6) + 1e-6)
    # values exactly on the grid round-trip exactly (lo, hi themselves are on the grid)
    v = np.array([-1.0, 1.0, 0.0, 0.2 * 1, -0.25, 0.5, 0.5, 0.5], np.float16)
    cb2 = np.array([-1.0, -0.25, 0.0, 0.5, 1.0, 1.5, 2.0, 3.0], np.float32)
    codes, idx, val, s, z = O.quantize_value(v, 0, cb2)
    assert (s, z) == (1.0, 0.0)
    on_grid = [0, 1, 2, 4, 5, 6, 7]
    assert np.array_equal(cb2[codes[on_grid]].astype(np.float16), v[on_grid])


def test_value_degenerate_range():
    cb = np.array([-1.0, -0.5, 0.5, 1.0], np.float32)
    v = np.full(16, 2.5, np.float16)
    codes, idx, val, s, z = O.quantize_value(v, 0, cb)
    assert s == 0.0 and z == 2.5 and np.all(codes == 0)


# ---------------------------------------------------------------------- packing --
def test_packing_golden(golden):
    for c in golden("packing.json")["cases"]:
        w = O.pack(np.array(c["codes"]), c["bits"])
        assert w.tolist() == c["words"]
        assert O.unpack(w, len(c["codes"]), c["bits"]).tolist() == c["codes"]


def test_packing_roundtrip_and_size():
    rng = np.random.default_rng(4)
    for bits in (2, 3, 4):
        for n in (0, 1, 8, 33, 1000):
            codes = rng.integers(0, 1 << bits, n)
            w = O.pack(codes, bits)
            assert w.size == (n * bits + 31) // 32
            assert np.array_equal(O.unpack(w, n, bits), codes)


# --------------------------------------------------------------------- attention --
def _all_fp16_codebook():
    """Every finite fp16 value (-0 folded into +0), strictly ascending (reading R19)."""
    allv = np.arange(65536, dtype=np.uint32).astype(np.uint16).view(np.float16)
    allv = allv[np.isfinite(allv)].astype(np.float64)
    return np.unique(allv).astype(np.float32)   # unique folds -0 and +0


def _textbook_attention(K, V, q, pos, H_q, H_kv, d, pos_base=0):
    """numpy fp64, HF rotate_half RoPE, softmax(q~ k~ / sqrt d) V."""
    T = K.shape[0]
    half = d // 2
    inv = 10000.0 ** (-np.arange(half) * 2.0 / d)

    def rot(x, p):
        ang = np.outer(p, inv)
        cos = np.concatenate([np.cos(ang)] * 2, axis=-1)
        sin = np.concatenate([np.sin(ang)] * 2, axis=-1)
        rh = np.concatenate([-x[..., half:], x[..., :half]], axis=-1)
        return x * cos + rh * sin

    G = H_q // H_kv
    out = np.zeros((H_q, d))
    Kf, Vf, qf = K.astype(np.float64), V.astype(np.float64), q.astype(np.float64)
    for g in range(H_q):
        h = g // G
        kr = rot(Kf[:, h * d:(h + 1) * d], np.arange(T) + pos_base)
        qr = rot(qf[g][None], np.array([pos]))[0]
        s = kr @ qr / np.sqrt(d)
        p = np.exp(s - s.max())
        out[g] = p @ Vf[:, h * d:(h + 1) * d] / p.sum()
    return out


@pytest.mark.parametrize("H_q,H_kv", [(1, 1), (2, 2), (4, 2)])
def test_attention_lossless_equals_textbook(H_q, H_kv):
    d, T = 8, 6
    D = H_kv * d
    rng = np.random.default_rng(H_q * 10 + H_kv)
    K = (rng.standard_normal((T, D)) * 0.6).astype(np.float16)   # some beyond [-1,1] -> outliers
    V = (rng.standard_normal((T, D)) * 3).astype(np.float16)
    q = rng.standard_normal((H_q, d)).astype(np.float16)
    cb = _all_fp16_codebook()
    lo, hi = -np.ones(D, np.float32), np.ones(D, np.float32)
    cache = O.prefill(K, V, lo, hi, cb, cb, ppm=0, value_identity_affine=True)
    o = O.attend(cache, q, 41, H_q=H_q, H_kv=H_kv, d=d, key_lo=lo, key_hi=hi,
                 cbK_dec=cb, cbV_dec=cb, pos_base=36)
    ref = _textbook_attention(K, V, q, 41, H_q, H_kv, d, pos_base=36)
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-12)


def test_attention_lossless_matches_torch_sdpa():
    torch = pytest.importorskip("torch")
    d, T, H = 8, 5, 2
    rng = np.random.default_rng(7)
    K = (rng.standard_normal((T, H * d)) * 0.5).astype(np.float16)
    V = rng.standard_normal((T, H * d)).astype(np.float16)
    q = rng.standard_normal((H, d)).astype(np.float16)
    cb = _all_fp16_codebook()
    lo, hi = -np.ones(H * d, np.float32), np.ones(H * d, np.float32)
    cache = O.prefill(K, V, lo, hi, cb, cb, ppm=0, value_identity_affine=True)
    o = O.attend(cache, q, T - 1, H_q=H, H_kv=H, d=d, key_lo=lo, key_hi=hi, cbK_dec=cb, cbV_dec=cb)
    # torch: HF-style rotate_half RoPE + SDPA in fp64 (library routine)
    half = d // 2
    inv = 1.0 / (10000.0 ** (torch.arange(0, d, 2, dtype=torch.float64) / d))

    def rot(x, p):
        ang = torch.outer(p.double(), inv)
        emb = torch.cat([ang, ang], -1)
        rh = torch.cat([-x[..., half:], x[..., :half]], -1)
        return x * emb.cos() + rh * emb.sin()

    Kt = torch.tensor(K.astype(np.float64)).view(T, H, d).transpose(0, 1)
    Vt = torch.tensor(V.astype(np.float64)).view(T, H, d).transpose(0, 1)
    qt = torch.tensor(q.astype(np.float64))[:, None, :]
    kr = rot(Kt, torch.arange(T))
    qr = rot(qt, torch.tensor([T - 1]))
    ref = torch.nn.functional.scaled_dot_product_attention(qr, kr, Vt)[:, 0, :].numpy()
    np.testing.assert_allclose(o, ref, rtol=1e-10, atol=1e-12)


def test_attention_selection_and_uniform():
    d, T, H = 8, 7, 1
    rng = np.random.default_rng(9)
    K = (rng.standard_normal((T, d)) * 0.5).astype(np.float16)
    V = rng.standard_normal((T, d)).astype(np.float16)
    cb = np.linspace(-1, 1, 16).astype(np.float32)
    lo, hi = -np.ones(d, np.float32), np.ones(d, np.float32)
    cache = O.prefill(K, V, lo, hi, cb, cb, ppm=125_000)
    kw = dict(H_q=1, H_kv=1, d=d, key_lo=lo, key_hi=hi, cbK_dec=cb, cbV_dec=cb)
    # uniform: q = 0 -> every score 0 -> o = mean of dequantized V
    o0 = O.attend(cache, np.zeros((1, d), np.float16), 3, **kw)
    deqV = cb[cache.vcodes].astype(np.float64) * cache.vs[:, None] + cache.vz[:, None]
    for n in range(T):
        for r, c in enumerate(cache.vidx[n]):
            deqV[n, c] = np.float64(cache.vval[n, r].view(np.float16))
    np.testing.assert_allclose(o0[0], deqV.mean(axis=0), rtol=1e-12, atol=1e-12)
    # q = 0: every score is exactly 0, so m = 0 and l = T (the selection pin with a
    # dominant score is test_selection_one_dominant_token_returns_its_dequantized_value)
    p = O.attend_partial(cache, np.zeros((1, d), np.float16), 3, **kw)
    assert p[0, d + 1] == T and p[0, d] == 0.0


# ------------------------------------------------ hand-computed attention pins ------
def _cb4():
    return np.array([-1.0, -0.5, 0.5, 1.0], np.float32)


def test_score_d2_one_token_quantized_key_by_hand():
    """S:506 (qk_scores example): d=2, one token, key quantized with a NON-identity
    per-channel affine, score computed by hand.

    key_lo = [0, -2], key_hi = [2, 4]  ->  s_c = (hi-lo)/2 = [1, 3], z_c = (hi+lo)/2 = [1, 1]
    (reading R6).  x = [1.25, 0.25]: normalised (x-z)/s = [0.25, -0.25] -> nearest
    centroids of [-1,-.5,.5,1] are 0.5 and -0.5 (codes 2, 1), so
    K^ = [0.5*1 + 1, -0.5*3 + 1] = [1.5, -0.5]   (Chat[code]*s + z).
    q = [2, 1].  With pos == pos_base + n both sides get the same rotation, so
    q~.k~ = q.K^ = 2*1.5 - 0.5 = 2.5 and s = 2.5/sqrt(2).  With pos - n = 1 (theta_0 = 1
    for d=2) q~ = R(1) q and q~.K^ = 2.5 (cos 1 - sin 1).  A slip in the Key
    dequantization (cb*s - z, (cb+z)*s, s and z swapped) changes both numbers.
    """
    lo, hi = np.array([0.0, -2.0], np.float32), np.array([2.0, 4.0], np.float32)
    K = np.array([[1.25, 0.25]], np.float16)
    V = np.array([[1.0, 3.0]], np.float16)
    cache = O.prefill(K, V, lo, hi, _cb4(), _cb4(), ppm=0)
    assert list(cache.kcodes[0]) == [2, 1] and cache.kidx.size == 0
    kw = dict(H_q=1, H_kv=1, d=2, key_lo=lo, key_hi=hi, cbK_dec=_cb4(), cbV_dec=_cb4())
    q = np.array([[2.0, 1.0]], np.float16)
    p = O.attend_partial(cache, q, 7, pos_base=7, **kw)
    assert abs(p[0, 2] - 2.5 / np.sqrt(2.0)) < 1e-12 and p[0, 3] == 1.0
    cos1, sin1 = 0.5403023058681398, 0.8414709848078965   # tests/golden/rope.json d=2 n=1
    p = O.attend_partial(cache, q, 1, pos_base=0, **kw)
    assert abs(p[0, 2] - 2.5 * (cos1 - sin1) / np.sqrt(2.0)) < 1e-12


def test_selection_one_dominant_token_returns_its_dequantized_value():
    """S:515 (av_matvec example "w one-hot at token t -> out == dequantized V_t") through
    attend: a query aligned with token 1's key at fp16 scale 6e4 makes its score exceed
    the others by > 1e6, so o == V^_1 exactly.

    V_1 = [0.5, 3.0, 1.0, 2.5]: lo = 0.5, hi = 3 -> s_n = 1.25, z_n = 1.75; normalised
    [-1, 1, -0.6, 0.6] -> codes [0, 3, 1, 2] -> V^_1 = [0.5, 3.0, 1.125, 2.375]
    (Chat*s_n + z_n; per-token affine).
    Keys: lo = -8, hi = 8 (s = 8, z = 0); token 1 = +8 everywhere, tokens 0, 2 = -8.
    pos = pos_base + 1, so token 1 sees no relative rotation: score_1 = 4*6e4*8/2 = 9.6e5,
    while score_0, score_2 = -q.R(+-1)K^_1/2 < 0.
    """
    lo, hi = np.full(4, -8.0, np.float32), np.full(4, 8.0, np.float32)
    K = np.array([[-8.0] * 4, [8.0] * 4, [-8.0] * 4], np.float16)
    V = np.array([[-3.0, 7.0, 0.5, 2.0], [0.5, 3.0, 1.0, 2.5], [4.0, -1.0, 6.0, 0.0]], np.float16)
    cache = O.prefill(K, V, lo, hi, _cb4(), _cb4(), ppm=0)
    assert list(cache.vcodes[1]) == [0, 3, 1, 2]
    assert cache.vs[1] == 1.25 and cache.vz[1] == 1.75
    kw = dict(H_q=1, H_kv=1, d=4, key_lo=lo, key_hi=hi, cbK_dec=_cb4(), cbV_dec=_cb4())
    q = np.full((1, 4), 60000.0, np.float16)
    p = O.attend_partial(cache, q, 11, pos_base=10, **kw)
    assert abs(p[0, 4] - 960000.0) < 1e-6 and p[0, 5] == 1.0
    o = O.attend(cache, q, 11, pos_base=10, **kw)
    assert list(o[0]) == [0.5, 3.0, 1.125, 2.375]


def test_uniform_scores_mean_of_hand_dequantized_values():
    """q = 0 gives uniform weights (every score 0), so o = mean of V^ (S:516 convexity).
    V_0 = [0.5, 3, 1, 2.5] -> V^_0 = [0.5, 3, 1.125, 2.375] (see the selection pin).
    V_1 = [-2, 2, 0, 1]: s = 2, z = 0, normalised [-1, 1, 0, 0.5]; 0 is equidistant from
    -0.5 and 0.5 and the tie goes to the lower index (R8) -> codes [0, 3, 1, 2] ->
    V^_1 = [-2, 2, -1, 1].  Mean = [-0.75, 2.5, 0.0625, 1.6875]."""
    lo, hi = np.full(4, -8.0, np.float32), np.full(4, 8.0, np.float32)
    K = np.array([[1.0, -2.0, 3.0, 0.5], [-1.0, 2.0, 5.0, 4.0]], np.float16)
    V = np.array([[0.5, 3.0, 1.0, 2.5], [-2.0, 2.0, 0.0, 1.0]], np.float16)
    cache = O.prefill(K, V, lo, hi, _cb4(), _cb4(), ppm=0)
    assert list(cache.vcodes[1]) == [0, 3, 1, 2]
    kw = dict(H_q=1, H_kv=1, d=4, key_lo=lo, key_hi=hi, cbK_dec=_cb4(), cbV_dec=_cb4())
    o = O.attend(cache, np.zeros((1, 4), np.float16), 5, **kw)
    assert list(o[0]) == [-0.75, 2.5, 0.0625, 1.6875]


def test_merge_any_partition_equals_unsplit():
    d, H, T = 8, 2, 23
    rng = np.random.default_rng(11)
    K = gen.gen_keys(0, 0, T, H * d)
    V = gen.gen_values(0, 0, T, H * d)
    q = rng.standard_normal((H, d)).astype(np.float16)
    cb = np.linspace(-1, 1, 8).astype(np.float32)
    lo = np.percentile(K.astype(np.float64), 2, axis=0).astype(np.float32)
    hi = np.percentile(K.astype(np.float64), 98, axis=0).astype(np.float32)
    full = O.prefill(K, V, lo, hi, cb, cb, ppm=62_500)
    kw = dict(H_q=H, H_kv=H, d=d, key_lo=lo, key_hi=hi, cbK_dec=cb, cbV_dec=cb)
    o_full = O.attend(full, q, T + 5, **kw)
    for cuts in ([0, 23], [0, 1, 23], [0, 10, 11, 23], [0, 5, 9, 17, 22, 23]):
        parts = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            sub = O.prefill(K[a:b], V[a:b], lo, hi, cb, cb, ppm=62_500)
            parts.append(O.attend_partial(sub, q, T + 5, pos_base=a, **kw))
        np.testing.assert_allclose(O.merge(np.stack(parts)), o_full, rtol=1e-12, atol=1e-13)


def test_prefill_equals_successive_appends():
    D = 16
    K = gen.gen_keys(1, 0, 9, D)
    V = gen.gen_values(1, 0, 9, D)
    cb = np.linspace(-1, 1, 8).astype(np.float32)
    lo, hi = np.full(D, -1.5, np.float32), np.full(D, 1.5, np.float32)
    full = O.prefill(K, V, lo, hi, cb, cb, ppm=125_000)
    for n in range(9):
        c, i, v = O.quantize_key(K[n], lo, hi, cb)
        assert np.array_equal(full.kcodes[n], c)
        assert np.array_equal(full.kidx[full.kptr[n]:full.kptr[n + 1]], i)
        c2, i2, v2, s, z = O.quantize_value(V[n], 125_000, cb)
        assert np.array_equal(full.vcodes[n], c2) and np.array_equal(full.vidx[n], i2)
        assert full.vs[n] == s and full.vz[n] == z


# ------------------------------------------------ online Key thresholds (f2) pins --
@pytest.mark.parametrize("T,D,ppm", [(97, 8, 10_000), (2048, 16, 10_000), (300, 4, 50_000), (50, 3, 0)])
def test_online_key_thresholds_order_statistics(T, D, ppm):
    """lo / hi = the floor(n/2)-th smallest and ceil(n/2)-th largest excluded -> numpy's sort
    (a library routine), and brute force: exactly ceil(n/2) values of the channel lie strictly
    above hi or tie into the excluded set, floor(n/2) below lo likewise."""
    rng = np.random.default_rng(T + D)
    K = (rng.standard_t(3, size=(T, D)) * 2.0).astype(np.float16)
    K[T // 3, 0] = np.float16(-0.0)
    lo, hi = O.key_thresholds_online(K, ppm)
    n = (ppm * T + 999_999) // 1_000_000
    ku, kl = (n + 1) // 2, n // 2
    srt = np.sort(K.astype(np.float64), axis=0)
    np.testing.assert_array_equal(lo, srt[kl].astype(np.float32) + 0.0)
    np.testing.assert_array_equal(hi, srt[T - 1 - ku].astype(np.float32) + 0.0)
    for c in range(D):
        x = K[:, c].astype(np.float64)
        assert (x > hi[c]).sum() <= ku and (x >= hi[c]).sum() >= ku + 1
        assert (x < lo[c]).sum() <= kl and (x <= lo[c]).sum() >= kl + 1
    # the worked example of S:328-333 read per channel: {2, 4} excluded, kept range [-0.2, 0.3]
    v = np.array([0.1, -0.2, 5.0, 0.3, -4.0, 0.0], np.float16)[:, None]
    lo1, hi1 = O.key_thresholds_online(v, 333_333)   # ceil(6 f) = 2
    assert float(lo1[0]) == float(np.float16(-0.2)) and float(hi1[0]) == float(np.float16(0.3))
