"""C-ABI boundary checks that need no GPU (-m "not gpu").

The library must load on a CPU-only box, export every symbol include/kvq.h declares,
and reject invalid configurations synchronously (validation runs before any CUDA
call, so these return KVQ_EINVAL / KVQ_ESHAPE without a device).
"""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvq():
    from paper_2401_18079_b200._build import build
    build()
    from paper_2401_18079_b200 import kvq as m
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kvq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kvq_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    syms = declared_symbols()
    for s in ("kvq_cache_create", "kvq_append", "kvq_prefill_quantize", "kvq_decode_attend"):
        assert s in syms


def test_library_exports_every_declared_symbol(kvq):
    lib = kvq.lib()
    syms = declared_symbols()
    assert sorted(kvq.EXPORTED) == syms
    for s in syms:
        assert hasattr(lib, s), s
    assert kvq.version() >= 100
    assert lib.kvq_last_error() is not None


def test_library_has_sm100a_code():
    import subprocess
    from paper_2401_18079_b200._build import LIB
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _args(D=256, bits=3, nlev=None):
    nlev = nlev or (1 << bits)
    cb = np.linspace(-1, 1, nlev).astype(np.float32)
    return dict(n_q_heads=D // 128, n_kv_heads=D // 128, head_dim=128, bits=bits,
                outlier_ppm=10_000, capacity_tokens=64, key_cb=cb, val_cb=cb,
                key_lo=-np.ones(D, np.float32), key_hi=np.ones(D, np.float32))


@pytest.mark.parametrize("patch,status", [
    (dict(bits=5), 1), (dict(bits=1), 1), (dict(outlier_ppm=500_000), 1),
    (dict(outlier_ppm=-1), 1), (dict(head_dim=64), 2), (dict(capacity_tokens=0), 1),
    (dict(n_q_heads=3), 2), (dict(rope_theta=-1.0), 1),
])
def test_create_rejects_invalid_config(kvq, patch, status):
    a = _args()
    a.update(patch)
    with pytest.raises(kvq.KVQError) as e:
        kvq.KVQCache(**a)
    assert e.value.status == status


def test_create_rejects_bad_codebooks_and_thresholds(kvq):
    a = _args()
    a["key_cb"] = np.array([0, 0, 1, 2, 3, 4, 5, 6], np.float32)      # not strictly ascending
    with pytest.raises(kvq.KVQError) as e:
        kvq.KVQCache(**a)
    assert e.value.status == kvq.KVQ_EINVAL
    a = _args()
    a["key_lo"] = np.ones(256, np.float32) * 2                         # lo > hi
    with pytest.raises(kvq.KVQError):
        kvq.KVQCache(**a)
    a = _args()
    a["val_cb"] = np.array([0, 1, 2, np.nan, 4, 5, 6, 7], np.float32)
    with pytest.raises(kvq.KVQError):
        kvq.KVQCache(**a)
