"""Seeded synthetic workloads for KVQuant decode attention (inputs only).

This package holds the input generators shared by the oracle side and the CUDA side
(tests/, bench.py, smoke) plus the offline calibration tooling that turns calibration
tokens into the constants ``kvq_cache_create`` takes.  It contains none of the hot
path's arithmetic (quantize / dequantize / RoPE / attend).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import calib, gen  # noqa: F401


@dataclass(frozen=True)
class Workload:
    name: str
    n_layers: int
    H_q: int
    H_kv: int
    d: int
    T: int
    bits: int
    ppm: int = 10_000          # 1% outliers
    qnorm: bool = False

    @property
    def D(self) -> int:
        return self.H_kv * self.d


# BASELINE.json "configs" (index = config number - 1).
CONFIGS = {
    "c1": Workload("c1-1L-1H-d128-4K-nuq4-1%", 1, 1, 1, 128, 4096, 4),
    "c2": Workload("c2-llama7b-1L-32K-nuq3-1%", 1, 32, 32, 128, 32768, 3),
    "c3_nuq4": Workload("c3-llama7b-32L-128K-nuq4-1%", 32, 32, 32, 128, 131072, 4),
    "c3_nuq3": Workload("c3-llama7b-32L-128K-nuq3-1%", 32, 32, 32, 128, 131072, 3),
    "c4": Workload("c4-mistral7b-32L-1M-nuq3-1%", 32, 32, 8, 128, 1 << 20, 3),
    "c5": Workload("c5-llama7b-10M-nuq2-1%-qnorm", 32, 32, 32, 128, 10_000_000, 2, qnorm=True),
}

# Not BASELINE configs: the other paper models the attend kernels tile, for extra
# measurements only (bench.py --workload NAME).
EXTRA_CONFIGS = {
    "c4_nuq4": Workload("x-mistral7b-32L-1M-nuq4-1%", 32, 32, 8, 128, 1 << 20, 4),
    "l70b": Workload("x-llama2-70b-80L-128K-nuq3-1%", 80, 64, 8, 128, 131072, 3),
}


def calibrate(seed: int, layer: int, D: int, bits: int, ppm: int, n_cal: int = 4096,
              qnorm: bool = False):
    """Generate calibration tokens for one layer and run offline calibration."""
    Kc = gen.gen_keys(seed, layer, n_cal, D, stream=gen.STREAM_CAL_K)
    Vc = gen.gen_values(seed, layer, n_cal, D, stream=gen.STREAM_CAL_V)
    return calib.calibrate_layer(Kc, Vc, bits, ppm, qnorm=qnorm)
