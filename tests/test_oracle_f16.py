"""Pins of the oracle's fp16-comparator functions (BASELINE config C3's fp16 cache; P:598,
P:608): each is checked against a library routine or an exact special case, not against
itself.  CPU only."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")


def test_f64_to_f16_matches_numpy_rne():
    """IEEE round-to-nearest-even: numpy's float64 -> float16 conversion (one rounding)."""
    rng = np.random.default_rng(0)
    xs = [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, -65520.0, 1e9, 6e-8, 5.96e-8,
          2.98e-8, 2.99e-8, 6.1e-5, 6.097e-5, 1.5, 2049.0, 2051.0, 3.0e-5]
    xs += list(rng.normal(0, 1, 2000)) + list(rng.normal(0, 3000, 1000)) + list(rng.normal(0, 1e-5, 1000))
    # exact ties between consecutive fp16 values (normal and subnormal): even mantissa wins
    h = rng.integers(0, 0x7bff, 500).astype(np.uint16)
    lo = h.view(np.float16).astype(np.float64)
    hi = (h + 1).view(np.float16).astype(np.float64)
    xs += list((lo + hi) / 2) + list(-(lo + hi) / 2)
    for x in xs:
        assert O.f64_to_f16(x) == int(np.float64(x).astype(np.float16).view(np.uint16)), x


def test_f16cache_key_is_rounded_rope():
    rng = np.random.default_rng(1)
    H, d = 3, 128
    k = rng.normal(0, 4, H * d).astype(np.float16)
    for pos in (0, 1, 777, 9_999_999):
        st = O.f16cache_keys(k[None], H, d, pos_base=pos)[0]
        ref = np.concatenate([O.rope(k[h * d:(h + 1) * d].astype(np.float64), pos) for h in range(H)])
        np.testing.assert_array_equal(st, ref.astype(np.float16).view(np.uint16))
        if pos == 0:   # RoPE at position 0 is the identity: the stored Key is the input
            np.testing.assert_array_equal(st, k.view(np.uint16))


def test_attend_dense_matches_torch_sdpa():
    rng = np.random.default_rng(2)
    H_q = H_kv = 4
    d, T, pos = 128, 300, 5000
    K = rng.normal(0, 1, (T, H_kv * d)).astype(np.float16)
    V = rng.normal(0, 1, (T, H_kv * d)).astype(np.float16)
    q = (rng.normal(0, 2, (H_q, d))).astype(np.float16)
    Kp = O.f16cache_keys(K, H_kv, d, pos_base=0)
    o = O.attend_dense(Kp, V, q, pos, H_q=H_q, H_kv=H_kv, d=d)
    qr = np.stack([O.rope(q[g].astype(np.float64), pos) for g in range(H_q)])
    Kt = torch.from_numpy(Kp.view(np.float16).astype(np.float64)).reshape(T, H_kv, d).permute(1, 0, 2)
    Vt = torch.from_numpy(V.astype(np.float64)).reshape(T, H_kv, d).permute(1, 0, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(torch.from_numpy(qr)[:, None, :], Kt, Vt)[:, 0, :]
    np.testing.assert_allclose(o, ref.numpy(), rtol=0, atol=1e-12)
