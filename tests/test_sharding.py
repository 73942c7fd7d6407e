"""Sequence-sharding host logic with world_size-2 gloo on CPU (-m "not gpu").

Each rank quantizes its token shard with pos_base = its start (oracle side: the oracle is
test infrastructure; the product's merge runs on the GPU), gathers the partials with the
product's gather_partials over gloo, and the rank-ordered log-sum-exp merge of the
gathered partials must equal the unsharded attention on every rank, bitwise identical
across ranks.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, result_dir):
    sys.path.insert(0, ROOT)
    import oracle as O
    from kvq_synth import calib, gen
    from paper_2401_18079_b200.sharding import ShardPlan, gather_partials

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, D, ppm = 2, 256, 10_000
    cal = calib.calibrate_layer(gen.gen_keys(0, 0, 512, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(0, 0, 512, D, stream=gen.STREAM_CAL_V), 3, ppm)
    K, V = gen.gen_keys(0, 0, T, D), gen.gen_values(0, 0, T, D)
    q = gen.gen_queries(0, 0, H, H, 128)[0]
    plan = ShardPlan(T, world, rank)
    a, b = plan.start, plan.end
    sub = O.prefill(K[a:b], V[a:b], cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
    part = O.attend_partial(sub, q, T + 3, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"],
                            key_hi=cal["key_hi"], cbK_dec=cal["cbK"], cbV_dec=cal["cbV"],
                            pos_base=plan.pos_base)
    parts = gather_partials(torch.from_numpy(part))
    o = O.merge(parts.numpy())
    np.save(os.path.join(result_dir, f"o{rank}.npy"), o)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [97, 256])
def test_gloo_world2_sharded_equals_unsharded(tmp_path, T):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, T, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    o0, o1 = np.load(tmp_path / "o0.npy"), np.load(tmp_path / "o1.npy")
    assert np.array_equal(o0, o1)            # bitwise identical on every rank
    import oracle as O
    from kvq_synth import calib, gen
    H, D, ppm = 2, 256, 10_000
    cal = calib.calibrate_layer(gen.gen_keys(0, 0, 512, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(0, 0, 512, D, stream=gen.STREAM_CAL_V), 3, ppm)
    K, V = gen.gen_keys(0, 0, T, D), gen.gen_values(0, 0, T, D)
    q = gen.gen_queries(0, 0, H, H, 128)[0]
    full = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], ppm)
    ref = O.attend(full, q, T + 3, H_q=H, H_kv=H, d=128, key_lo=cal["key_lo"],
                   key_hi=cal["key_hi"], cbK_dec=cal["cbK"], cbV_dec=cal["cbV"])
    np.testing.assert_allclose(o0, ref, rtol=1e-12, atol=1e-13)


def test_shard_plan_ranges():
    from paper_2401_18079_b200.sharding import ShardPlan
    for T in (1, 7, 100, 10_000_000):
        for world in (1, 2, 4, 8):
            rngs = [ShardPlan(T, world, r).range_of(r) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == T
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
            assert ShardPlan(T, world, world - 1).capacity(5) == rngs[-1][1] - rngs[-1][0] + 5
            assert ShardPlan(T, world, 0).pos_base == 0
