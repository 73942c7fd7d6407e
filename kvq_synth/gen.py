"""Seeded synthetic inputs (no method arithmetic) -- shared by the oracle side and the
CUDA side of every parity test, and by bench.py.

Recipe (after PAPER.md fig:activation-distribution P:243-255,
fig:percentiles P:737-749):
  Keys (pre-RoPE), per layer: channel c has sigma_c = 1 for 97% of channels and
    sigma_c ~ U[8, 24] for 3% "outlier channels" (chosen by a seeded permutation);
    mu_c = 0.5 * sigma_c * N(0,1); x = mu_c + sigma_c * (N(0,1) + spike),
    spike = +-(3 + 5U) with probability 1.5%.
  Values: x = rho_n * (N(0,1) + spike), rho_n = exp(0.3 N(0,1)),
    spike = +-(4 + 8U) with probability 1% ("no fixed outlier pattern").
  Queries: N(0,1) * q_scale with q_scale chosen from the key variance so the score
    standard deviation is about 2.
Everything is rounded to fp16 (the paper's baseline dtype).

CPU generator: numpy Philox (counter-based), keyed by (seed, stream, layer).
GPU generator (bench only, large configs): torch.cuda generator with the same recipe;
its values are not bit-identical to the CPU ones (bench inputs need no oracle parity).
"""
from __future__ import annotations

import numpy as np

STREAM_K, STREAM_V, STREAM_Q, STREAM_CAL_K, STREAM_CAL_V, STREAM_APP_K, STREAM_APP_V, STREAM_PARAM = range(1, 9)

F16_MAX = 65504.0


def rng(seed: int, stream: int, layer: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[(int(seed) << 16) ^ int(stream), int(layer) + 1]))


def _to_f16(x: np.ndarray) -> np.ndarray:
    return np.clip(x, -F16_MAX, F16_MAX).astype(np.float16)


def key_channel_params(seed: int, layer: int, D: int):
    """Per-channel (mu_c, sigma_c) of the synthetic pre-RoPE Keys."""
    g = rng(seed, STREAM_PARAM, layer)
    sigma = np.ones(D, dtype=np.float64)
    n_out = max(1, int(round(0.03 * D)))
    chans = g.permutation(D)[:n_out]
    sigma[chans] = g.uniform(8.0, 24.0, size=n_out)
    mu = 0.5 * sigma * g.standard_normal(D)
    return mu, sigma


def gen_keys(seed: int, layer: int, T: int, D: int, stream: int = STREAM_K) -> np.ndarray:
    mu, sigma = key_channel_params(seed, layer, D)
    g = rng(seed, stream, layer)
    z = g.standard_normal((T, D))
    u = g.random((T, D))
    spike_on = g.random((T, D)) < 0.015
    sign = np.where(g.random((T, D)) < 0.5, -1.0, 1.0)
    spike = np.where(spike_on, sign * (3.0 + 5.0 * u), 0.0)
    return _to_f16(mu[None, :] + sigma[None, :] * (z + spike))


def gen_values(seed: int, layer: int, T: int, D: int, stream: int = STREAM_V) -> np.ndarray:
    g = rng(seed, stream, layer)
    rho = np.exp(0.3 * g.standard_normal((T, 1)))
    z = g.standard_normal((T, D))
    u = g.random((T, D))
    spike_on = g.random((T, D)) < 0.01
    sign = np.where(g.random((T, D)) < 0.5, -1.0, 1.0)
    spike = np.where(spike_on, sign * (4.0 + 8.0 * u), 0.0)
    return _to_f16(rho * (z + spike))


def query_scale(seed: int, layer: int, D: int, d: int) -> np.ndarray:
    """Per-KV-head query scale so that q.k/sqrt(d) has std ~2 (from the key recipe)."""
    mu, sigma = key_channel_params(seed, layer, D)
    e_spike2 = 0.015 * (9.0 + 15.0 + 25.0 / 3.0)
    ek2 = mu ** 2 + sigma ** 2 * (1.0 + e_spike2)
    per_head = ek2.reshape(-1, d).mean(axis=1)
    return 2.0 / np.sqrt(per_head)


def gen_queries(seed: int, layer: int, H_q: int, H_kv: int, d: int, n: int = 1) -> np.ndarray:
    """[n, H_q, d] fp16 queries (pre-RoPE)."""
    g = rng(seed, STREAM_Q, layer)
    sc = query_scale(seed, layer, H_kv * d, d)
    G = H_q // H_kv
    scale = np.repeat(sc, G)[None, :, None]
    return _to_f16(g.standard_normal((n, H_q, d)) * scale)


# ---------------------------------------------------------------- GPU generator ---
def gen_layer_torch(seed: int, layer: int, T: int, D: int, device, which: str,
                    param_seed: int = 0, param_layer: int = 0):
    """Large-config generator on the GPU (bench only).  Same recipe, torch RNG; the
    per-channel Key statistics come from (param_seed, param_layer) so they match the
    calibration tokens of that layer."""
    import torch

    mu, sigma = key_channel_params(param_seed, param_layer, D)
    gen = torch.Generator(device=device)
    gen.manual_seed((seed * 1000003 + layer * 7919 + (1 if which == "K" else 2)) & 0x7FFFFFFFFFFF)
    out = torch.empty((T, D), dtype=torch.float16, device=device)
    chunk = max(1, (1 << 26) // D)
    mu_t = torch.tensor(mu, dtype=torch.float32, device=device)
    sg_t = torch.tensor(sigma, dtype=torch.float32, device=device)
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        n = t1 - t0
        z = torch.randn((n, D), generator=gen, device=device)
        u = torch.rand((n, D), generator=gen, device=device)
        on = torch.rand((n, D), generator=gen, device=device)
        sgn = torch.where(torch.rand((n, D), generator=gen, device=device) < 0.5, -1.0, 1.0)
        if which == "K":
            spike = torch.where(on < 0.015, sgn * (3.0 + 5.0 * u), torch.zeros_like(u))
            x = mu_t[None, :] + sg_t[None, :] * (z + spike)
        else:
            rho = torch.exp(0.3 * torch.randn((n, 1), generator=gen, device=device))
            spike = torch.where(on < 0.01, sgn * (4.0 + 8.0 * u), torch.zeros_like(u))
            x = rho * (z + spike)
        out[t0:t1] = x.clamp_(-F16_MAX, F16_MAX).to(torch.float16)
    return out
