"""Host-side multi-rank logic on CPU with gloo, world_size 2 and 4 (-m "not gpu").

Covers the sharding maps (every global trajectory exactly once, inputs of a
shard = the slice of the global inputs), and the two exchange steps of
paper_2304_06835_b200.multi_gpu (all-gather of statistics triples, gather of
states to rank 0). The merge itself is a CUDA kernel tested on the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_06835_b200 import multi_gpu as mg
from synth.inputs import make_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # statistics exchange: rank r contributes triples filled with r
        local = torch.full((2, 3, 3), float(rank + 1), dtype=torch.float64)
        g = mg.allgather_stats(local)
        assert g.shape == (world, 2, 3, 3)
        for r in range(world):
            assert torch.all(g[r] == r + 1)
        # state gather to rank 0
        st = torch.arange(12, dtype=torch.float32).reshape(3, 4) + 100 * rank
        out = mg.gather_states(st, dst=0)
        if rank == 0:
            assert out.shape == (world, 3, 4)
            for r in range(world):
                assert torch.equal(out[r], torch.arange(12, dtype=torch.float32).reshape(3, 4) + 100 * r)
        else:
            assert out is None
        # each rank's shard inputs equal the slice of the global ensemble
        N_total = world * 4096
        for sh in [mg.shard_contiguous(N_total, rank, world), mg.shard_block_cyclic(N_total, rank, world, chunk=512)]:
            u0, p = make_inputs("lorenz", "random10", sh.n_local, seed=0xC5, index_offset=sh.index_offset,
                                chunk_len=sh.chunk_len, chunk_stride=sh.chunk_stride)
            ug, pg = make_inputs("lorenz", "random10", N_total, seed=0xC5)
            gi = sh.global_indices().numpy()
            assert np.array_equal(p, pg[:, gi]) and np.array_equal(u0, ug[:, gi])
        # bench.py's workloads: C5 strong scaling splits N_total contiguously (every global index
        # exactly once, shard sizes within one), C2 weak scaling gives every rank N per GPU
        import bench

        class A:
            workload, n_total, traj_per_gpu = "c5", 10**8 + 3, 7
        sh, Nt = bench.workload_sizes(A, rank, world)
        parts = [None] * world
        dist.all_gather_object(parts, (sh.index_offset, sh.n_local))
        assert Nt == A.n_total and sum(n for _, n in parts) == Nt
        off = 0
        for o, n in parts:
            assert o == off
            off += n
        assert max(n for _, n in parts) - min(n for _, n in parts) <= 1
        A.workload = "c2"
        sh, Nt = bench.workload_sizes(A, rank, world)
        assert Nt == 7 * world and sh.index_offset == 7 * rank and sh.n_local == 7
        # a C5 shard's on-device inputs are the slice of the global ensemble (host twin, small N_total)
        A.workload, A.n_total = "c5", world * 1000 + 1
        sh, Nt = bench.workload_sizes(A, rank, world)
        u0, p = make_inputs("lorenz", "random10", sh.n_local, seed=0xC5, index_offset=sh.index_offset, N_total=Nt,
                            dtype="f32")
        ug, pg = make_inputs("lorenz", "random10", Nt, seed=0xC5, dtype="f32")
        lo = sh.index_offset
        assert np.array_equal(p, pg[:, lo:lo + sh.n_local]) and np.array_equal(u0, ug[:, lo:lo + sh.n_local])
        # multi_gpu.solve rejects inconsistent layouts before any device work
        for kw, msg in [(dict(shard="block_cyclic", gather="peer"), "contiguous"),
                        (dict(shard="diagonal"), "unknown shard"),
                        (dict(gather="allgather"), "unknown gather")]:
            with pytest.raises(ValueError, match=msg):
                mg.solve("lorenz", "tsit5", "random10", world * 4096, (0.0, 1.0), 1e-3, device="cpu", **kw)
        with pytest.raises(ValueError, match="equal shards"):
            mg.solve("lorenz", "tsit5", "random10", world * 4096 + 1, (0.0, 1.0), 1e-3, gather="nccl", device="cpu")
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


@pytest.mark.parametrize("N,R", [(10**8, 8), (10**7 + 3, 4), (5, 2), (1 << 20, 8)])
def test_shards_cover_every_index_once(N, R):
    for maker in [mg.shard_contiguous, lambda n, r, w: mg.shard_block_cyclic(n, r, w, chunk=1 << 16)]:
        shards = [maker(N, r, R) for r in range(R)]
        assert sum(s.n_local for s in shards) == N
        if N <= 1 << 20:
            allidx = np.concatenate([s.global_indices().numpy() for s in shards])
            assert np.array_equal(np.sort(allidx), np.arange(N))
    w = [mg.shard_weak(1000, r, 4) for r in range(4)]
    assert [s.index_offset for s in w] == [0, 1000, 2000, 3000]
