"""GPU parity of the fp16 comparator cache (kvq_f16_*; BASELINE config C3's fp16 arm, the
paper's fp16 mat-vec baseline P:598) against the oracle (kvo_f16cache_key,
kvo_attend_dense).  Stored Keys: RoPE(k) rounded once to fp16; the GPU's fp64 sin/cos may
differ from glibc's by an ulp, which can move a value sitting on an fp16 rounding boundary by
one fp16 ulp, so the stored Keys must be bit-exact except for at most 1e-4 of the elements,
which must be within one ulp.  Values bit-exact.  Attention within 1e-3 (fp32 accumulation)."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import TOL_FP32, rel_err_per_head

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = TOL_FP32


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


@pytest.mark.parametrize("H,T,base", [(1, 77, 0), (8, 1000, 0), (32, 2113, 0), (8, 700, 9_990_000)])
def test_f16_cache_store_and_attend(kvq, H, T, base):
    D = H * 128
    K = gen.gen_keys(51, 0, T, D)
    V = gen.gen_values(51, 0, T, D)
    c = kvq.F16Cache(n_q_heads=H, n_kv_heads=H, capacity_tokens=T + 8, pos_base=base)
    c.append(torch.from_numpy(K[: T // 2]).cuda(), torch.from_numpy(V[: T // 2]).cuda())
    c.append(K[T // 2:], V[T // 2:])                      # host buffers are staged
    kst, vst = c.export()
    kref = O.f16cache_keys(K, H, 128, pos_base=base)
    np.testing.assert_array_equal(vst, V.view(np.uint16))
    diff = kst.astype(np.int32) - kref.astype(np.int32)
    assert np.abs(diff).max() <= 1 and np.count_nonzero(diff) <= max(1, kst.size // 10_000)
    for k, pos in enumerate((base + T - 1, base + T + 4321)):
        q = gen.gen_queries(52 + k, 0, H, H, 128)[0]
        o = torch.zeros((H, 128), dtype=torch.float32, device="cuda")
        c.attend(torch.from_numpy(q).cuda(), pos, o)
        torch.cuda.synchronize()
        exp = O.attend_dense(kref, V, q, pos, H_q=H, H_kv=H, d=128)
        err = rel_err_per_head(o.cpu().numpy(), exp)
        assert err.max() < TOL, err


def test_f16_cache_errors(kvq):
    c = kvq.F16Cache(n_q_heads=2, n_kv_heads=2, capacity_tokens=4)
    q = torch.zeros((2, 128), dtype=torch.float16, device="cuda")
    o = torch.zeros((2, 128), dtype=torch.float32, device="cuda")
    with pytest.raises(kvq.KVQError) as e:
        c.attend(q, 0, o)
    assert e.value.status == kvq.KVQ_EEMPTY
    K = torch.zeros((5, 256), dtype=torch.float16, device="cuda")
    with pytest.raises(kvq.KVQError) as e:
        c.append(K, K)
    assert e.value.status == kvq.KVQ_ECAPACITY
    with pytest.raises(kvq.KVQError) as e:
        kvq.F16Cache(n_q_heads=4, n_kv_heads=2, capacity_tokens=4)
    assert e.value.status == kvq.KVQ_ESHAPE
