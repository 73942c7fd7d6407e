"""Chunk-paged sequences on the GPU: sequences grown from a shared pool of
fixed-size chunk caches, attended in one batched-partial launch over all chunks and merged per
sequence, against the oracle on each whole sequence; chunks reused by a later sequence at other
positions."""
import numpy as np
import pytest

import oracle as O
from kvq_synth import gen

from .gpu_common import make_cache, rel_err_per_head, setup_layer, tol_attend

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


@pytest.mark.parametrize("H_q,H_kv,bits", [(8, 8, 3), (8, 2, 3), (8, 8, 2)])
def test_paged_sequences_match_oracle(kvq, H_q, H_kv, bits):
    from paper_2401_18079_b200.paged import ChunkPool, PagedSequence, attend_paged
    ppm, chunk = 10_000, 128
    cal, _, _ = setup_layer(61, 0, H_q, H_kv, bits, ppm, 8)
    D = H_kv * 128
    pool = ChunkPool(8, chunk, lambda cap: make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=cap))

    def run(specs):
        seqs, refs, qs, outs, poss = [], [], [], [], []
        for i, (pos_base, n_pre, n_app) in enumerate(specs):
            n = n_pre + n_app
            K, V = gen.gen_keys(62 + i, 0, n, D), gen.gen_values(62 + i, 0, n, D)
            s = PagedSequence(pool, pos_base=pos_base)
            s.prefill(torch.from_numpy(K[:n_pre]).cuda(), torch.from_numpy(V[:n_pre]).cuda())
            for t in range(n_pre, n):
                s.append(torch.from_numpy(K[t]).cuda(), torch.from_numpy(V[t]).cuda())
            seqs.append(s)
            refs.append(O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm))
            qs.append(torch.from_numpy(gen.gen_queries(70 + i, 0, H_q, H_kv, 128)[0]).cuda())
            outs.append(torch.zeros((H_q, 128), dtype=torch.float32, device="cuda"))
            poss.append(pos_base + n + 3)
        attend_paged(seqs, qs, poss, outs)
        torch.cuda.synchronize()
        for i, (pos_base, _, _) in enumerate(specs):
            exp = O.attend(refs[i], qs[i].cpu().numpy(), poss[i], H_q=H_q, H_kv=H_kv, d=128,
                           key_lo=cal["key_lo"], key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"],
                           cbV_dec=cal["cbV_dec"], pos_base=pos_base)
            err = rel_err_per_head(outs[i].cpu().numpy(), exp)
            assert err.max() < tol_attend(H_q, H_kv, bits), (i, err)
        return seqs

    # A spans 3 chunks (300 prefill + 5 appends: 128, 128, 49), B one partial chunk, C exactly 2
    seqs = run([(0, 300, 5), (0, 100, 0), (2000, 256, 0)])
    assert [len(s.chunks) for s in seqs] == [3, 1, 2]
    assert pool.free_chunks == 2
    for s in seqs:
        s.release()
    assert pool.free_chunks == 8
    # the reset chunks serve new sequences at other positions
    run([(10_000, 130, 2), (7, 60, 1)])
