"""batched decode (kvq_decode_attend_batch): B independent sequences with
their own caches and lengths in ONE launch (the warp-autonomous MHA kernel, or the tensor-core
GQA kernel for G = 2, 4, 8), each output against the oracle on its own cache."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import TOL_ATTEND, make_cache, rel_err_per_head, setup_layer, tol_attend

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


@pytest.mark.parametrize("H_q,H_kv,bits,lens", [(8, 8, 3, [33, 1000, 4096, 100, 1, 2500, 64, 777]),
                                                (8, 8, 4, [300, 31, 1500]),
                                                (8, 8, 2, [32, 2049]),
                                                (32, 8, 3, [200, 513, 64]),
                                                (8, 4, 2, [100, 1, 700, 33]),
                                                (16, 2, 3, [300, 64, 2048]),
                                                (8, 2, 4, [129, 1000])])
def test_batched_decode_matches_oracle(kvq, H_q, H_kv, bits, lens):
    ppm = 10_000
    cal, _, _ = setup_layer(81, 0, H_q, H_kv, bits, ppm, 8)
    caches, refs, qs, outs, poss = [], [], [], [], []
    D = H_kv * 128
    Kall, Vall = gen.gen_keys(81, 0, sum(lens), D), gen.gen_values(81, 0, sum(lens), D)
    offs = np.cumsum([0] + lens)
    for i, T in enumerate(lens):
        K, V = Kall[offs[i]:offs[i + 1]], Vall[offs[i]:offs[i + 1]]
        c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 4, pos_base=1000 * i)
        c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
        caches.append(c)
        refs.append(O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm))
        q = gen.gen_queries(90 + i, 0, H_q, H_kv, 128)[0]
        qs.append(torch.from_numpy(q).cuda())
        outs.append(torch.zeros((H_q, 128), dtype=torch.float32, device="cuda"))
        poss.append(1000 * i + T + i)
    kvq.attend_batch(caches, qs, poss, outs)
    torch.cuda.synchronize()
    for i in range(len(lens)):
        exp = O.attend(refs[i], qs[i].cpu().numpy(), poss[i], H_q=H_q, H_kv=H_kv, d=128, key_lo=cal["key_lo"],
                       key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"], pos_base=1000 * i)
        err = rel_err_per_head(outs[i].cpu().numpy(), exp)
        assert err.max() < tol_attend(H_q, H_kv, bits), (i, err)
    expected_kernel = 2 if H_q != H_kv else 1
    assert all(c.info()["attend_kernel"] == expected_kernel for c in caches)
    # the same step again (tickets reset, scratch reused) gives the same result
    outs2 = [torch.zeros_like(o) for o in outs]
    kvq.attend_batch(caches, qs, poss, outs2)
    torch.cuda.synchronize()
    for a, b in zip(outs, outs2):
        assert torch.equal(a, b)


def test_batched_decode_errors(kvq):
    cal, K, V = setup_layer(83, 0, 8, 8, 3, 10_000, 64)
    a = make_cache(kvq, cal, 8, 8, 3, 10_000, capacity=64)
    b = make_cache(kvq, cal, 8, 8, 3, 10_000, capacity=64)
    a.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    q = torch.zeros((8, 128), dtype=torch.float16, device="cuda")
    o = [torch.zeros((8, 128), dtype=torch.float32, device="cuda") for _ in range(2)]
    with pytest.raises(kvq.KVQError) as e:
        kvq.attend_batch([a, b], [q, q], [64, 64], o)
    assert e.value.status == kvq.KVQ_EEMPTY
