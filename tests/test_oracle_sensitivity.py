"""Pins for the oracle's mixed-precision pieces (-m "not gpu").

Fisher diagonal, the sensitivity Omega of eq:opt2, the one-shot
assignment and the dequantization they rest on.
Worked values come from SPEC's sensitivity module (hand arithmetic) or are derived by hand
below; the rest are closed forms, invariants and brute force.
"""
import itertools

import numpy as np
import pytest

import oracle as O
from tests.test_oracle_pins import _all_fp16_codebook


# ------------------------------------------------------------------- Fisher diagonal --
def test_fisher_diag_spec_examples():
    # SPEC sensitivity/fisher_diag: [[1,2],[3,-1]] -> [10, 5]; zero gradient; single square
    np.testing.assert_array_equal(O.fisher_diag([[1, 2], [3, -1]]), [10.0, 5.0])
    np.testing.assert_array_equal(O.fisher_diag([[0, 0, 0]]), [0.0, 0.0, 0.0])
    np.testing.assert_array_equal(O.fisher_diag([[2]]), [4.0])


def test_fisher_diag_errors_and_order():
    with pytest.raises(ValueError):
        O.fisher_diag([])
    with pytest.raises(ValueError):
        O.fisher_diag([[1, 2], [1, 2, 3]])
    rng = np.random.default_rng(3)
    g = rng.integers(-50, 50, size=(7, 13)).astype(np.float64)   # integers: sums are exact
    F = O.fisher_diag(list(g))
    np.testing.assert_array_equal(F, O.fisher_diag(list(g[::-1])))   # permutation invariant
    np.testing.assert_array_equal(F, (g ** 2).sum(0))
    assert (F >= 0).all()


# --------------------------------------------------------------- sensitivity Omega ----
def test_layer_sensitivity_spec_examples():
    # SPEC: a=[1,2], qa=[1,1.5], f=[10,5] -> 10*0 + 5*0.25 = 1.25
    assert O.layer_sensitivity([1, 2], [1, 1.5], [10, 5]) == 1.25
    assert O.layer_sensitivity([1, 2], [1, 2], [10, 5]) == 0.0          # qa == a
    assert O.layer_sensitivity([1, 2], [7, -3], [0, 0]) == 0.0          # f = 0
    assert O.layer_sensitivity([1, 2], [1, 1.5]) == 0.25                 # F = 1: squared error
    with pytest.raises(ValueError):
        O.layer_sensitivity([1, 2], [1, 2, 3])


def test_layer_sensitivity_linear_in_f():
    rng = np.random.default_rng(5)
    a, qa = rng.standard_normal(64), rng.standard_normal(64)
    f = rng.random(64)
    w = O.layer_sensitivity(a, qa, f)
    assert O.layer_sensitivity(a, qa, 4 * f) == pytest.approx(4 * w, rel=1e-15)
    f2 = rng.random(64)
    assert O.layer_sensitivity(a, qa, f + f2) == pytest.approx(w + O.layer_sensitivity(a, qa, f2), rel=1e-14)


# ------------------------------------------------------------------ assignment ---------
def test_assign_spec_examples():
    assert O.assign_mixed_precision([5, 1, 3], 1) == [1]
    assert O.assign_mixed_precision([5, 1, 3], 0) == []
    assert O.assign_mixed_precision([2, 2, 2], 2) == [0, 1]            # ties -> lower id
    with pytest.raises(ValueError):
        O.assign_mixed_precision([1, 2], 3)


def test_assign_brute_force_and_scaling():
    rng = np.random.default_rng(11)
    for L in range(1, 7):
        om = rng.random(L)
        for k in range(L + 1):
            got = O.assign_mixed_precision(om, k)
            # brute force: the unique k-subset of minimal total sensitivity (distinct omegas)
            best = min(itertools.combinations(range(L), k), key=lambda s: sum(om[i] for i in s))
            assert got == sorted(best)
            assert O.assign_mixed_precision(om * 37.5, k) == got       # argsort invariance


# ------------------------------------------------------- dequantize / layer Omega ------
CB2 = np.array([-1.0, -0.5, 0.5, 1.0], np.float32)


def test_layer_omega_hand_example():
    """D = 4, T = 1, 2-bit codebook [-1, -0.5, 0.5, 1].
    Keys, every channel lo = -2, hi = 2 (s = 2, z = 0):
      x = 1.25 -> 0.625 -> nearest 0.5 -> K^ = 1.0, error 0.25;  x = 3 > hi -> outlier, exact;
      x = -2 -> -1 -> K^ = -2 exact;  x = 0.5 -> 0.25 -> ties? |0.25-0.5| = 0.25 < 0.75 -> 0.5
      -> K^ = 1.0, error -0.5.   Omega_K = 0.0625 + 0.25 = 0.3125.
    Values v = [0.5, -1, 4, 0], ppm 250000 -> k = 1 outlier, the largest (R3): channel 2.
      Kept range [-1, 0.5] -> s = 0.75, z = -0.25:  0.5 -> 1 -> exact;  -1 -> -1 -> exact;
      0 -> 1/3 -> nearest 0.5 -> V^ = 0.125, error -0.125.   Omega_V = 0.015625."""
    K = np.array([[1.25, 3.0, -2.0, 0.5]], np.float16)
    V = np.array([[0.5, -1.0, 4.0, 0.0]], np.float16)
    lo, hi = np.full(4, -2.0, np.float32), np.full(4, 2.0, np.float32)
    ok, ov = O.layer_omega(K, V, lo, hi, CB2, CB2, 250_000)
    assert ok == 0.3125
    assert ov == 0.015625
    # Fisher weights select single terms
    FK = np.array([[0, 0, 0, 3]], np.float64)
    FV = np.array([[9, 9, 9, 8]], np.float64)
    ok, ov = O.layer_omega(K, V, lo, hi, CB2, CB2, 250_000, FK=FK, FV=FV)
    assert ok == 0.75 and ov == 0.125
    # decode codebook differs from encode (Q-Norm, R9): K^ uses the decode entries
    dec = np.array([-1.0, -0.5, 0.25, 1.0], np.float32)
    Kh, Vh = O.dequantize(O.prefill(K, V, lo, hi, CB2, CB2, 250_000), lo, hi, dec, dec)
    np.testing.assert_array_equal(Kh[0], [0.5, 3.0, -2.0, 0.5])
    np.testing.assert_array_equal(Vh[0], [1.0 * 0.75 - 0.25, -1.0, 4.0, 0.25 * 0.75 - 0.25])


def test_layer_omega_lossless_is_zero():
    # every fp16 value a codebook entry, Keys within [-1, 1] or outliers, identity Value affine
    rng = np.random.default_rng(2)
    K = (rng.standard_normal((6, 8)) * 0.6).astype(np.float16)
    V = (rng.standard_normal((6, 8)) * 3).astype(np.float16)
    cb = _all_fp16_codebook()
    lo, hi = -np.ones(8, np.float32), np.ones(8, np.float32)
    cache = O.prefill(K, V, lo, hi, cb, cb, ppm=0, value_identity_affine=True)
    Kh, Vh = O.dequantize(cache, lo, hi, cb, cb)
    np.testing.assert_array_equal(Kh, K.astype(np.float64))
    np.testing.assert_array_equal(Vh, V.astype(np.float64))


def test_dequantize_values_equal_single_token_attention():
    # with one cached token softmax is 1, so the pinned attend returns V^_0 for every head
    rng = np.random.default_rng(9)
    d, H = 8, 2
    D = H * d
    K = rng.standard_normal((1, D)).astype(np.float16)
    V = (rng.standard_normal((1, D)) * 2).astype(np.float16)
    lo, hi = np.full(D, -1.5, np.float32), np.full(D, 1.5, np.float32)
    cache = O.prefill(K, V, lo, hi, CB2, CB2, ppm=70_000)
    _, Vh = O.dequantize(cache, lo, hi, CB2, CB2)
    o = O.attend(cache, rng.standard_normal((H, d)).astype(np.float16), 3, H_q=H, H_kv=H, d=d,
                 key_lo=lo, key_hi=hi, cbK_dec=CB2, cbV_dec=CB2)
    np.testing.assert_allclose(o.reshape(-1), Vh[0], rtol=0, atol=1e-15)


def test_lower_precision_is_more_sensitive():
    # the quantization error at 2 bits exceeds that at 4 bits (uniform grids)
    rng = np.random.default_rng(4)
    K = rng.standard_normal((40, 16)).astype(np.float16)
    V = rng.standard_normal((40, 16)).astype(np.float16)
    lo, hi = np.full(16, -2.5, np.float32), np.full(16, 2.5, np.float32)
    om = {}
    for b in (2, 4):
        cb = np.linspace(-1, 1, 2 ** b).astype(np.float32)
        om[b] = sum(O.layer_omega(K, V, lo, hi, cb, cb, 62_500))
    assert om[2] > 2 * om[4] > 0
