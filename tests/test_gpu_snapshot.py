"""Cache snapshot / restore (SURVEY 5 checkpoint / resume): a restored cache
equals the original (canonical export, bit-identical attention) and continues exactly as it
would (further appends and attends); a snapshot of another configuration is refused."""
import numpy as np
import pytest

from kvq_synth import gen

from .gpu_common import make_cache, setup_layer

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_18079_b200 import kvq as m
    return m


def _same_export(a, b):
    ea, eb = a.export(), b.export()
    for k in ea:
        np.testing.assert_array_equal(ea[k], eb[k], k)


@pytest.mark.parametrize("H_q,H_kv,bits,T", [(8, 8, 3, 333), (8, 2, 3, 130), (8, 8, 4, 64)])
def test_snapshot_restore_roundtrip(kvq, H_q, H_kv, bits, T):
    ppm = 10_000
    cal, K, V = setup_layer(91, 0, H_q, H_kv, bits, ppm, T + 40)
    a = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 64)
    a.prefill(torch.from_numpy(K[:T - 5]).cuda(), torch.from_numpy(V[:T - 5]).cuda())
    for t in range(T - 5, T):
        a.append(torch.from_numpy(K[t]).cuda(), torch.from_numpy(V[t]).cuda())
    snap = a.snapshot()
    b = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=T + 64)
    b.prefill(torch.from_numpy(K[:7]).cuda(), torch.from_numpy(V[:7]).cuda())   # replaced by restore
    b.restore(snap)
    assert b.num_tokens == T
    _same_export(a, b)
    q = torch.from_numpy(gen.gen_queries(92, 0, H_q, H_kv, 128)[0]).cuda()
    oa = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
    ob = torch.zeros_like(oa)
    a.attend(q, T + 2, oa)
    b.attend(q, T + 2, ob)
    torch.cuda.synchronize()
    assert torch.equal(oa, ob)
    # both continue identically
    for t in range(T, T + 40):
        for c in (a, b):
            c.append(torch.from_numpy(K[t]).cuda(), torch.from_numpy(V[t]).cuda())
    a.attend(q, T + 45, oa)
    b.attend(q, T + 45, ob)
    torch.cuda.synchronize()
    assert torch.equal(oa, ob)
    _same_export(a, b)


def test_restore_refuses_other_configuration(kvq):
    ppm = 10_000
    cal3, K, V = setup_layer(93, 0, 8, 8, 3, ppm, 64)
    a = make_cache(kvq, cal3, 8, 8, 3, ppm, capacity=128)
    a.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    snap = a.snapshot()
    cal2, _, _ = setup_layer(93, 0, 8, 8, 2, ppm, 8)
    b = make_cache(kvq, cal2, 8, 8, 2, ppm, capacity=128)
    with pytest.raises(kvq.KVQError):
        b.restore(snap)
    small = make_cache(kvq, cal3, 8, 8, 3, ppm, capacity=32)
    with pytest.raises(kvq.KVQError):
        small.restore(snap)
    with pytest.raises(kvq.KVQError):
        a.restore(snap[:100])
