"""Sequence sharding through the PRODUCT path with two processes (verdict r1
item 7): both ranks share cuda:0, each quantizes its token shard into its own cache (pos_base =
shard start) with kvq_prefill_quantize, computes kvq_decode_attend_partial on the GPU,
exchanges the [H_q][d+2] partials through gloo on host copies (the product's
gather_partials), and merges them with kvq_merge_partials on the GPU.  The merged o must be
bitwise identical on both ranks and within the attention tolerance of the unsharded oracle."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H_q, H_kv, bits, T, result_dir):
    sys.path.insert(0, ROOT)
    from kvq_synth import gen
    from paper_2401_18079_b200 import kvq
    from paper_2401_18079_b200.sharding import ShardPlan, gather_partials
    from tests.gpu_common import make_cache, setup_layer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ppm = 10_000
    cal, K, V = setup_layer(61, 0, H_q, H_kv, bits, ppm, T)
    q = gen.gen_queries(62, 0, H_q, H_kv, 128)[0]
    plan = ShardPlan(T, world, rank)
    a, b = plan.start, plan.end
    c = make_cache(kvq, cal, H_q, H_kv, bits, ppm, capacity=b - a, pos_base=plan.pos_base)
    c.prefill(torch.from_numpy(K[a:b]).cuda(), torch.from_numpy(V[a:b]).cuda())
    part = torch.zeros((H_q, 130), dtype=torch.float32, device="cuda")
    c.attend_partial(torch.from_numpy(q).cuda(), T + 7, part)
    torch.cuda.synchronize()
    parts = gather_partials(part.cpu())                 # gloo, host copies
    o = torch.zeros((H_q, 128), dtype=torch.float32, device="cuda")
    kvq.merge_partials(parts.cuda(), o)
    torch.cuda.synchronize()
    np.save(os.path.join(result_dir, f"o{rank}.npy"), o.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H_q,H_kv,bits,T", [(8, 8, 3, 1000), (32, 8, 3, 777), (2, 2, 4, 300)])
def test_two_process_sharded_partials_product_path(tmp_path, H_q, H_kv, bits, T):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import oracle as O
    from kvq_synth import gen
    from tests.gpu_common import rel_err_per_head, setup_layer

    mp.spawn(_worker, args=(2, _free_port(), H_q, H_kv, bits, T, str(tmp_path)), nprocs=2, join=True)
    o0 = np.load(tmp_path / "o0.npy")
    o1 = np.load(tmp_path / "o1.npy")
    np.testing.assert_array_equal(o0.view(np.uint32), o1.view(np.uint32))
    ppm = 10_000
    cal, K, V = setup_layer(61, 0, H_q, H_kv, bits, ppm, T)
    q = gen.gen_queries(62, 0, H_q, H_kv, 128)[0]
    ref = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
    exp = O.attend(ref, q, T + 7, H_q=H_q, H_kv=H_kv, d=128, key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                   cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"])
    from tests.gpu_common import TOL_ATTEND
    assert rel_err_per_head(o0, exp).max() < TOL_ATTEND
