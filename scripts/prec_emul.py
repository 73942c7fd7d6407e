"""Numerical emulation of the attend kernels' score arithmetic (diagnostic, CPU only).

Builds a layer with the oracle, dequantizes K^ / V^ exactly (fp64), and recomputes the
attention output with the kernel's roundings switched on one at a time:
  table  : the fp16 (A, B) pair-table entries (scaled so the largest non-heavy entry is 2^14)
  cs16   : cos/sin of the token angle as the kernel forms them in fp16 (anchor x table, HMUL2 +
           HFMA2) or, 'cs16_1r', rounded once from the exact value
  heavy  : the largest-bound pairs (<= 8 per head, > 1/2 of the head max) kept exact (fp32)
  w16    : P.V weights p s_n 2^(14-E) rounded to fp16 (E per 32-token tile)
and reports the per-head max relative error against the exact fp64 result.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from kvq_synth import gen  # noqa: E402
from tests.gpu_common import setup_layer  # noqa: E402

LOG2E = 1.4426950408889634


def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def dequant(cache, cal, D):
    T = cache.T
    s = (cal["key_hi"].astype(np.float64) - cal["key_lo"]) / 2
    z = (cal["key_hi"].astype(np.float64) + cal["key_lo"]) / 2
    s = s.astype(np.float32).astype(np.float64)
    z = z.astype(np.float32).astype(np.float64)
    Kd = cal["cbK_dec"].astype(np.float64)[cache.kcodes] * s[None] + z[None]
    Kdense = Kd.copy()
    for n in range(T):
        a, b = cache.kptr[n], cache.kptr[n + 1]
        Kd[n, cache.kidx[a:b]] = cache.kval[a:b].view(np.float16).astype(np.float64)
    Vd = cal["cbV_dec"].astype(np.float64)[cache.vcodes] * cache.vs[:, None].astype(np.float64) + cache.vz[:, None].astype(np.float64)
    for n in range(T):
        Vd[n, cache.vidx[n]] = cache.vval[n].view(np.float16).astype(np.float64)
    return Kd, Kdense, Vd


def run(H_q, H_kv, bits, T, seed=4, kind=None, pos=None, variants=None):
    ppm = 10_000
    cal, K, V = setup_layer(seed, 0, H_q, H_kv, bits, ppm, T)
    if kind == "flat_values":
        V = V.astype(np.float32)
        rng = np.random.default_rng(31)
        for n in rng.choice(T, size=T // 3, replace=False):
            V[n, :] = np.float32(rng.normal())
        V = V.astype(np.float16)
    cache = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
    D = H_kv * 128
    Kd, Kdense, Vd = dequant(cache, cal, D)
    q = gen.gen_queries(seed, 0, H_q, H_kv, 128)[0].astype(np.float64)
    pos = T - 1 if pos is None else pos
    G = H_q // H_kv
    th = 10000.0 ** (-2.0 * np.arange(64) / 128)
    n = np.arange(T)
    ang_q = pos * th
    ang = n[:, None] * th[None]           # token angles
    res = {}
    for g in range(H_q):
        h = g // G
        qa, qb = q[g, :64], q[g, 64:]
        c, s = np.cos(ang_q), np.sin(ang_q)
        qt_a = (qa * c - qb * s) * LOG2E / np.sqrt(128)
        qt_b = (qb * c + qa * s) * LOG2E / np.sqrt(128)
        xa, xb = Kd[:, h * 128:h * 128 + 64], Kd[:, h * 128 + 64:h * 128 + 128]
        da, db = Kdense[:, h * 128:h * 128 + 64], Kdense[:, h * 128 + 64:h * 128 + 128]
        A = qt_a * xa + qt_b * xb
        B = qt_b * xa - qt_a * xb
        Ad = qt_a * da + qt_b * db          # dense-code table entries
        Bd = qt_b * da - qt_a * db
        cos, sin = np.cos(ang), np.sin(ang)
        s_exact = (A * cos + B * sin).sum(1)
        # heavy pairs: bound over codebook range ends
        cbK = cal["cbK_dec"].astype(np.float64)
        sK = ((cal["key_hi"].astype(np.float64) - cal["key_lo"]) / 2)[h * 128:h * 128 + 128]
        zK = ((cal["key_hi"].astype(np.float64) + cal["key_lo"]) / 2)[h * 128:h * 128 + 128]
        mx = np.maximum(np.abs(cbK[0] * sK + zK), np.abs(cbK[-1] * sK + zK))
        bound = np.maximum(np.abs(qt_a) * mx[:64] + np.abs(qt_b) * mx[64:], np.abs(qt_b) * mx[:64] + np.abs(qt_a) * mx[64:])
        tau = 0.5 * bound.max()
        while (bound > tau).sum() > 8:
            tau *= 1.25
        heavy = bound > tau
        rest = bound[~heavy].max()
        e = 14 - int(np.floor(np.log2(rest))) - 1
        sc = 2.0 ** e
        # cos/sin the kernel's way: tile anchor (n0 = 32 t) x cis(j th) in fp16
        n0 = (n // 32) * 32
        j = n % 32
        ac, as_ = f16(np.cos(n0[:, None] * th)), f16(np.sin(n0[:, None] * th))
        tc, ts = f16(np.cos(j[:, None] * th)), f16(np.sin(j[:, None] * th))
        c16 = f16(ac * tc)
        s16 = f16(as_ * tc)
        c16 = f16(-as_ * ts + c16)
        s16 = f16(ac * ts + s16)
        out = {}
        for name in variants:
            tab = "table" in name
            use_heavy = "heavy" in name
            if "cs16_1r" in name:
                cc, ss = f16(cos), f16(sin)
            elif "cs16" in name:
                cc, ss = c16, s16
            else:
                cc, ss = cos, sin
            Aq = f16(Ad * sc) / sc if tab else Ad
            Bq = f16(Bd * sc) / sc if tab else Bd
            if use_heavy:
                Aq = np.where(heavy[None], Ad, Aq)
                Bq = np.where(heavy[None], Bd, Bq)
                csx = np.where(heavy[None], cos, cc)
                snx = np.where(heavy[None], sin, ss)
            else:
                csx, snx = cc, ss
            corr = ((A - Ad) * cos + (B - Bd) * sin).sum(1)   # outlier terms (fp32 in the kernel)
            sc_ = (Aq * csx + Bq * snx).sum(1) + corr
            p = np.exp2(sc_ - sc_.max())
            if "w16" in name:
                sn = cache.vs.astype(np.float64)
                zn = cache.vz.astype(np.float64)
                cbV = cal["cbV_dec"].astype(np.float64)
                Vdn = cbV[cache.vcodes[:, h * 128:h * 128 + 128]]
                E = np.zeros(T)
                for t0 in range(0, T, 32):
                    smax = sn[t0:t0 + 32].max()
                    E[t0:t0 + 32] = np.floor(np.log2(smax)) + 1 if smax > 0 else 0
                w = f16(p * sn * 2.0 ** (14 - E)) * 2.0 ** (E - 14)
                ov = (w[:, None] * Vdn).sum(0) + (p * zn).sum()
                # outlier corrections exact
                dV = Vd[:, h * 128:h * 128 + 128] - (Vdn * sn[:, None] + zn[:, None])
                ov = ov + (p[:, None] * dV).sum(0)
                o = ov / p.sum()
            else:
                o = (p[:, None] * Vd[:, h * 128:h * 128 + 128]).sum(0) / p.sum()
            out[name] = o
        pe = np.exp2(s_exact - s_exact.max())
        oe = (pe[:, None] * Vd[:, h * 128:h * 128 + 128]).sum(0) / pe.sum()
        for name, o in out.items():
            res.setdefault(name, []).append(np.abs(o - oe).max() / np.abs(oe).max())
    return {k: (max(v), float(np.median(v))) for k, v in res.items()}


if __name__ == "__main__":
    V = ["table+cs16+heavy+w16", "table+cs16+heavy", "cs16+heavy", "table+heavy", "table",
         "table+cs16_1r+heavy", "table+cs16_1r+heavy+w16", "w16"]
    for cfg in [(2, 2, 4, 333), (32, 8, 3, 257), (8, 4, 3, 301), (32, 16, 3, 96), (40, 40, 3, 130)]:
        r = run(*cfg, variants=V)
        print(cfg, {k: "%.2e/%.1e" % v for k, v in r.items()})
    r = run(32, 8, 3, 161, seed=31, kind="flat_values", variants=V)
    print("flat", {k: "%.2e/%.1e" % v for k, v in r.items()})
