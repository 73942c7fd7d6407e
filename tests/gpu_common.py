"""Shared helpers for the GPU parity tests (oracle side vs CUDA side on the same seeded
inputs).  The oracle never sees anything produced by the CUDA path."""
from __future__ import annotations

import numpy as np

import oracle as O
from kvq_synth import calib, gen


def setup_layer(seed, layer, H_q, H_kv, bits, ppm, T, n_cal=2048, qnorm=False, d=128,
                fp16_codebooks=True):
    D = H_kv * d
    cal = calib.calibrate_layer(gen.gen_keys(seed, layer, n_cal, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(seed, layer, n_cal, D, stream=gen.STREAM_CAL_V),
                                bits, ppm, qnorm=qnorm, fp16_codebooks=fp16_codebooks)
    K = gen.gen_keys(seed, layer, T, D)
    V = gen.gen_values(seed, layer, T, D)
    return cal, K, V


def make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity, pos_base=0, device=0, **kw):
    return kvq.KVQCache(n_q_heads=H_q, n_kv_heads=H_kv, head_dim=128, bits=bits, outlier_ppm=ppm,
                        capacity_tokens=capacity, key_cb=cal["cbK"], val_cb=cal["cbV"],
                        key_cb_dec=cal["cbK_dec"], val_cb_dec=cal["cbV_dec"],
                        key_lo=cal["key_lo"], key_hi=cal["key_hi"], pos_base=pos_base,
                        device=device, **kw)


def assert_cache_equal(exp: dict, ref: O.CanonCache, t0: int = 0, t1: int | None = None):
    """Bit-exact comparison of a GPU export with the oracle's canonical cache."""
    t1 = ref.T if t1 is None else t1
    sl = slice(t0, t1)
    np.testing.assert_array_equal(exp["kcodes"].astype(np.uint16), ref.kcodes[sl], "key codes")
    np.testing.assert_array_equal(exp["vcodes"].astype(np.uint16), ref.vcodes[sl], "value codes")
    np.testing.assert_array_equal(exp["vs"].view(np.uint32), ref.vs[sl].view(np.uint32), "value scale")
    np.testing.assert_array_equal(exp["vz"].view(np.uint32), ref.vz[sl].view(np.uint32), "value offset")
    np.testing.assert_array_equal(exp["vidx"].astype(np.int32), ref.vidx[sl], "value outlier idx")
    np.testing.assert_array_equal(exp["vval"], ref.vval[sl], "value outlier val")
    kp = exp["kptr"] - exp["kptr"][0]
    rp = ref.kptr[t0:t1 + 1] - ref.kptr[t0]
    np.testing.assert_array_equal(kp, rp, "key CSC pointers")
    a, b = ref.kptr[t0], ref.kptr[t1]
    np.testing.assert_array_equal(exp["kidx"].astype(np.int32), ref.kidx[a:b], "key outlier idx")
    np.testing.assert_array_equal(exp["kval"], ref.kval[a:b], "key outlier val")


# Attention tolerances (reading R24).  north_star: "2e-3 max relative error, or
# 1e-3 when accumulating in fp32".  The quantized-cache kernels accumulate in fp32 but their
# products are fp16 by design (the paper's fp16 LUT arithmetic: fp16 K-table entries
# and fp16 rotation factors, each rounded once), so the fp16-arithmetic bar applies to them;
# their error is the designed arithmetic's (scripts/prec_emul.py reproduces it), and a median
# bound guards against regressions hiding under the max.  The fp16-cache comparator computes
# in fp32 and is held to 1e-3.
TOL_ATTEND = 2e-3
TOL_ATTEND_MEDIAN = 5e-4
TOL_FP32 = 1e-3


def tol_attend(H_q: int, H_kv: int, bits: int) -> float:
    """Per-head max tolerance of the attend kernel this configuration selects: the GQA kernel at
    2-4 bits (att_wgt_kernel) forms its Key scores from fp16 hi + lo operands on the tensor cores,
    i.e. fp32-accurate products, so it is held to the fp32 bar (R24); the LUT kernels to 2e-3."""
    return TOL_FP32 if (H_q != H_kv and bits in (2, 3, 4)) else TOL_ATTEND


def rel_err_per_head(o, ref):
    o = np.asarray(o, np.float64).reshape(ref.shape)
    num = np.abs(o - ref).max(axis=1)
    den = np.abs(ref).max(axis=1)
    return num / den


def merged_partial_to_natural(part):
    """Convert a GPU partial (m in log2 units) to the oracle's natural-log convention."""
    p = np.asarray(part, np.float64).copy()
    p[:, -2] = p[:, -2] * np.log(2.0)
    return p
