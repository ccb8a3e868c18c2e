"""multi_gpu.solve — the one-call multi-rank driver — on the one GPU of
this pool (-m gpu): two gloo ranks share cuda:0, so every step of the driver runs
(sharding, on-device inputs per shard, solve, stats all-gather + fixed-order merge,
fused peer gather or the collective gather). Rank 0 checks against one single-process
solve of the whole ensemble: states bit-identical (partition independence), merged
statistics equal to the single-process statistics within 1e-13 relative."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_2304_06835_b200 as ens
from paper_2304_06835_b200 import multi_gpu as mg
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)

def rel(a, b):
    return ((a - b).abs() / b.abs().clamp_min(1e-300)).max().item()

cases = [
    # (model, alg, recipe, N_total, tspan, dt, kw, shard, gather, saveat)
    ("lorenz", "tsit5", "random10", 6001, (0.0, 1.0), 1e-3, {}, "contiguous", "peer", None),
    ("lorenz", "tsit5", "rho_sweep", 8192, (0.0, 1.0), 1e-3,
     dict(adaptive=True, abstol=1e-6, reltol=1e-6), "block_cyclic", "nccl", None),
    ("lorenz", "vern7", "random10", 4000, (0.0, 1.0), 1e-3,
     dict(adaptive=True, abstol=1e-8, reltol=1e-8), "contiguous", "peer", [0.0, 0.5, 1.0]),
    ("lorenz_sde_add", "em", "const", 4096, (0.0, 1.0), 1e-3, dict(seed=0xC4), "contiguous", None,
     [0.0, 0.5, 1.0]),
]
for (model, alg, recipe, NT, tspan, dt, kw, shard, gather, sa) in cases:
    for dtype in (torch.float32, torch.float64):
        r = mg.solve(model, alg, recipe, NT, tspan, dt, dtype=dtype, input_seed=0xC5, shard=shard, chunk=1024,
                     gather=gather, stats=True, saveat=sa, device=dev, **kw)
        assert (r.local.retcode == 0).all().item()
        if rank == 0:
            U0, P = ens.generate_inputs(model, recipe, NT, dtype=dtype, seed=0xC5, N_total=NT, device=dev)
            sde = alg == "em"
            ref = ens.solve(model, alg, U0, P, tspan, dt, saveat=sa, stats=sde, **kw)
            ref_st = ref.stats if sde else ens.ensemble_stats(ref.u if sa else ref.u.unsqueeze(0))
            assert r.stats[..., 0].eq(NT).all().item(), (model, alg)
            assert rel(r.stats[..., 1], ref_st[..., 1]) <= 1e-13, (model, alg, dtype)
            assert rel(r.stats[..., 2], ref_st[..., 2]) <= 1e-12, (model, alg, dtype)
            if gather == "peer":
                assert torch.equal(r.gathered, ref.u), (model, alg, dtype)
            elif gather == "nccl":
                for q in range(world):
                    sh = (mg.shard_block_cyclic(NT, q, world, 1024) if shard == "block_cyclic"
                          else mg.shard_contiguous(NT, q, world))
                    assert torch.equal(r.gathered[q], ref.u[..., sh.global_indices().to(dev)]), (model, alg, q)
        else:
            assert r.gathered is None
        dist.barrier()
print("MULTI_SOLVE_OK", rank, flush=True)
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_multi_solve_two_ranks_one_gpu():
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=400)[0] for p in procs]
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"MULTI_SOLVE_OK {r}" in o, o[-3000:]
