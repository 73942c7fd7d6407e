"""Pins for the oracle's offline-calibration pieces (-m "not gpu").

Weighted 1-D k-means for eq:fisher_kmeans, the normalized kept points it runs on
(P:321), Q-Norm (eq:qnorm P:355-358).  Worked values are SPEC's nuq module (hand
arithmetic / exhaustive partitions) or derived by hand below; the rest are closed forms
(k-means of a uniform density), brute force over contiguous partitions, and invariants.
"""
import itertools

import numpy as np
import pytest

import oracle as O


# ------------------------------------------------------------------ k-means ---------
def test_kmeans_spec_examples():
    c, _ = O.fisher_kmeans([-1, -0.9, 0.8, 1.0], [1, 1, 1, 1], 2)
    np.testing.assert_allclose(c, [-0.95, 0.9], rtol=0, atol=1e-15)
    c, _ = O.fisher_kmeans([-1, 0, 1], [1, 4, 2], 2)                  # clusters {-1, 0}, {1}
    np.testing.assert_allclose(c, [-0.2, 1.0], rtol=0, atol=1e-15)
    x, w = np.array([-1.0, 0, 1]), np.array([1.0, 4, 2])
    assert np.sum(w * (x - c[O.nearest_label(x, c)]) ** 2) == pytest.approx(0.8, abs=1e-15)


def test_nearest_label_ties_to_lower():
    cb = [-1.0, 0.0, 1.0]
    np.testing.assert_array_equal(O.nearest_label([0.4, 0.5, 0.51, -0.5, -2, 2], cb), [1, 1, 2, 0, 0, 2])


def _contiguous_optimum(x, w, k):
    """Exhaustive search over contiguous partitions of the sorted points (1-D optimum)."""
    o = np.argsort(x)
    x, w = x[o], w[o]
    best = (np.inf, None)
    for cuts in itertools.combinations(range(1, len(x)), k - 1):
        b = (0,) + cuts + (len(x),)
        cost, cent = 0.0, []
        for a, e in zip(b[:-1], b[1:]):
            m = np.sum(w[a:e] * x[a:e]) / np.sum(w[a:e])
            cost += np.sum(w[a:e] * (x[a:e] - m) ** 2)
            cent.append(m)
        if cost < best[0]:
            best = (cost, np.array(cent))
    return best


@pytest.mark.parametrize("seed", range(6))
def test_kmeans_well_separated_is_optimal(seed):
    # k well-separated clusters, one inside each initial bin [-1 + 2j/k, -1 + 2(j+1)/k]: Lloyd
    # from the bin centres (R27) reaches the global optimum of the exhaustive search
    rng = np.random.default_rng(seed)
    k = int(rng.integers(2, 5))
    centres = -1.0 + (2.0 * np.arange(k) + 1.0) / k + rng.uniform(-0.3, 0.3, k) / k
    x = np.concatenate([c + rng.uniform(-0.01, 0.01, int(rng.integers(1, 4))) for c in centres])
    w = rng.uniform(0.5, 2.0, x.size)
    c, _ = O.fisher_kmeans(x, w, k, max_iter=200, tol=0)
    _, opt = _contiguous_optimum(x, w, k)
    np.testing.assert_allclose(c, opt, rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_kmeans_fixed_point_by_brute_force(seed):
    # at convergence every centroid is the weighted mean of the points nearest to it (distance
    # argmin by brute force, ties to the lower index) or keeps its place when it has none
    rng = np.random.default_rng(seed)
    x = np.clip(rng.standard_normal(500) * 0.35, -1, 1)
    w = rng.exponential(1.0, x.size)
    c, n = O.fisher_kmeans(x, w, 8, max_iter=1000, tol=0)
    d = np.abs(x[:, None] - c[None, :])
    lab = np.argmin(d, axis=1)                       # first minimum = lower index
    for j in range(8):
        if np.any(lab == j):
            assert c[j] == pytest.approx(np.sum(w[lab == j] * x[lab == j]) / np.sum(w[lab == j]), abs=1e-14)


def test_kmeans_objective_non_increasing_and_weight_scaling():
    rng = np.random.default_rng(3)
    x = np.clip(rng.standard_normal(3000) * 0.4, -1, 1)
    w = rng.exponential(1.0, x.size)
    prev = np.inf
    for it in range(1, 12):
        c, n = O.fisher_kmeans(x, w, 8, max_iter=it, tol=0)
        assert n == it
        obj = np.sum(w * (x - c[O.nearest_label(x, c)]) ** 2)
        assert obj <= prev * (1 + 1e-12)
        prev = obj
    c1, _ = O.fisher_kmeans(x, w, 8, max_iter=30, tol=0)
    c2, _ = O.fisher_kmeans(x, 8.0 * w, 8, max_iter=30, tol=0)      # argmin invariance of eq. 2
    np.testing.assert_allclose(c1, c2, rtol=0, atol=1e-12)


def test_kmeans_uniform_density_closed_form():
    # k-means of the uniform density on [-1, 1] is the k equal-width bin centres
    x = (np.arange(20_000) + 0.5) / 10_000 - 1.0
    c, _ = O.fisher_kmeans(x, np.ones_like(x), 4, max_iter=200, tol=1e-12)
    np.testing.assert_allclose(c, [-0.75, -0.25, 0.25, 0.75], atol=1e-4)
    assert np.all(np.abs(c + c[::-1]) < 1e-4)                      # symmetric


def test_kmeans_fisher_weights_pull_centroids_inward():
    # SPEC: weights concentrated near 0 -> spacing near 0 tighter than near +-1
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, 20_000)
    c, _ = O.fisher_kmeans(x, 1.0 / (np.abs(x) + 0.1), 8, max_iter=200)
    gaps = np.diff(c)
    assert gaps[3] < gaps[0] and gaps[3] < gaps[-1]
    cu, _ = O.fisher_kmeans(x, np.ones_like(x), 8, max_iter=200)
    assert np.abs(c).max() < np.abs(cu).max()


def test_kmeans_empty_cluster_keeps_centroid():
    # all points in one bin: the other centroids stay at their initial bin centres
    c, _ = O.fisher_kmeans([0.9, 0.95], [1, 1], 4, max_iter=5)
    np.testing.assert_allclose(c, [-0.75, -0.25, 0.25, 0.925], atol=1e-15)


# --------------------------------------------------------------- normalized points ----
def test_key_points_spec_normalize_example():
    # SPEC normalize_vector: v = [0, 2, 4], lo = 0, hi = 4 -> [-1, 0, 1]; outside values dropped;
    # a zero-width channel contributes nothing (R27)
    K = np.array([[0, 5], [2, 5], [4, 5], [6, 5]], np.float16)
    x, w = O.calib_key_points(K, [0, 5], [4, 5], FK=np.array([[1, 9], [2, 9], [3, 9], [4, 9]], np.float32))
    np.testing.assert_array_equal(x, [-1.0, 0.0, 1.0])
    np.testing.assert_array_equal(w, [1.0, 2.0, 3.0])


def test_value_points_hand_example():
    # token [0.5, -1, 4, 0], ppm 250000 -> k = 1 outlier (the largest, R3); kept range [-1, 0.5]
    # -> s = 0.75, z = -0.25: points 1, -1, 1/3
    V = np.array([[0.5, -1, 4, 0], [3, 3, 3, 3]], np.float16)      # 2nd token: zero width, dropped
    x, w = O.calib_value_points(V, 250_000)
    np.testing.assert_allclose(x, [1.0, -1.0, 1.0 / 3.0], rtol=0, atol=1e-16)
    np.testing.assert_array_equal(w, [1, 1, 1])


def test_value_points_tie_rule():
    # ties among the largest values: the lower index is the outlier (R3), so the kept copy of
    # the tied value carries the weight of the HIGHER index
    V = np.array([[2, 1, 2, 0]], np.float16)
    FV = np.array([[10, 20, 30, 40]], np.float32)
    x, w = O.calib_value_points(V, 250_000, FV)                    # k = 1: index 0 removed
    np.testing.assert_array_equal(x, [0.0, 1.0, -1.0])              # kept range [0, 2]
    np.testing.assert_array_equal(w, [20, 30, 40])


# -------------------------------------------------------------------- Q-Norm ----------
def test_qnorm_spec_example():
    np.testing.assert_allclose(O.apply_qnorm([-1, 0, 1], 0, 1, 0.1, 0.8), [-1.375, -0.125, 1.125], atol=1e-15)
    np.testing.assert_allclose(O.apply_qnorm([-1, 0, 1], 0.2, 0.5, 0.2, 0.5), [-1, 0, 1], atol=1e-15)


def test_qnorm_restores_mean_and_std():
    # decoding the ENCODE labels with the Q-Norm'd codebook gives the pre-quantization moments
    rng = np.random.default_rng(8)
    x = np.clip(rng.standard_normal(5000) * 0.3 + 0.1, -1, 1)
    cb = np.array([-0.8, -0.2, 0.3, 0.9])
    dec = O.apply_qnorm(cb, *O.qnorm_stats(x, cb))
    q = dec[O.nearest_label(x, cb)]
    assert q.mean() == pytest.approx(x.mean(), abs=1e-12)
    assert q.std() == pytest.approx(x.std(), rel=1e-12)


def test_calibrate_layer_properties():
    rng = np.random.default_rng(1)
    K = (rng.standard_normal((300, 16)) * rng.uniform(0.5, 3, 16)).astype(np.float16)
    V = rng.standard_normal((300, 16)).astype(np.float16)
    cal = O.calibrate_layer(K, V, 2, 20_000, max_iter=50, qnorm=True)
    lo, hi = O.key_thresholds_online(K, 20_000)
    np.testing.assert_array_equal(cal["key_lo"], lo)
    np.testing.assert_array_equal(cal["key_hi"], hi)
    for key in ("cbK", "cbV", "cbK_dec", "cbV_dec"):
        cb = cal[key]
        assert cb.dtype == np.float32 and cb.size == 4 and np.all(np.diff(cb) > 0)
        np.testing.assert_array_equal(cb, cb.astype(np.float16).astype(np.float32))   # fp16 values (R23)
    assert np.all(np.abs(cal["cbK"]) <= 1) and np.all(np.abs(cal["cbV"]) <= 1)
