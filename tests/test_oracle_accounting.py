"""Byte accounting and offline-calibration tooling pins (-m "not gpu")."""
import numpy as np

from oracle import accounting as A
from kvq_synth import calib


def test_avg_bits_reproduce_paper_table(golden):
    g = golden("accounting.json")
    for bits, f, lo, hi in g["avg_bits_ranges"]:
        v = A.avg_bits(bits, f, g["D"], g["seq_len"])
        assert lo <= v <= hi, (bits, f, v)
    for bits, f, lo, hi in g["ratios"]:
        assert lo <= A.compression_ratio(bits, f, g["D"], g["seq_len"]) <= hi


def test_per_head_vector_reading_does_not_reproduce_table(golden):
    # Reading R1: with a per-head vector (D = 128) the printed ranges are missed.
    g = golden("accounting.json")
    v = A.avg_bits(4, 0.01, 128, g["seq_len"])
    assert not (4.32 <= v <= 4.35)


def test_fp16_size_formula():
    # 2*n*h*d*b*l elements; LLaMA-7B at 128K -> 2^36 bytes (reading R18)
    assert A.fp16_kv_bytes(1, 1, 1, 1, 1) == 4
    assert A.fp16_kv_bytes(32, 32, 128, 1, 131072) == 2 ** 36


def test_qnorm_and_kmeans_golden(golden):
    g = golden("qnorm_kmeans.json")
    q = g["qnorm"]
    out = calib.apply_qnorm(q["C"], q["mu1"], q["sigma1"], q["mu2"], q["sigma2"])
    np.testing.assert_allclose(out, q["out"], rtol=0, atol=1e-6)
    assert np.array_equal(calib.apply_qnorm(q["C"], 0.3, 2.0, 0.3, 2.0), np.float32(q["C"]))
    for c in g["kmeans"]:
        cent = calib.kmeans_1d(c["points"], c["weights"], c["k"])
        np.testing.assert_allclose(cent, c["centroids"], atol=1e-9)


def test_key_thresholds_two_sided():
    x = np.arange(100, dtype=np.float64)[:, None].repeat(3, axis=1)
    lo, hi = calib.key_thresholds(x.astype(np.float16), ppm=40_000)   # 4 outliers: 2 up, 2 down
    assert lo.tolist() == [2.0] * 3 and hi.tolist() == [97.0] * 3
