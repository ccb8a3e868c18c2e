"""Fused gather (multi_gpu.PeerGather, ens_options.out_ld) on the one GPU of
this pool (-m gpu): two processes — rank 0 owns the global state array, rank 1
writes its shard into it through a CUDA IPC mapping (peer stores; on a
multi-GPU node the same code path stores over NVLink). The gathered array
must equal a single-process solve of the whole ensemble bit for bit."""
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
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_2304_06835_b200 as ens
from paper_2304_06835_b200 import multi_gpu as mg
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
N_total, k = 5000, 3
sa = [0.0, 0.5, 1.0]
for dt in (torch.float32, torch.float64):
    sh = mg.shard_contiguous(N_total, rank, world)
    u0, p = ens.generate_inputs("lorenz", "random10", sh.n_local, dtype=dt, seed=0xC5, index_offset=sh.index_offset,
                                N_total=N_total)
    pg = mg.PeerGather((k, 3), sh.n_local, sh.index_offset, N_total, dt, dev)
    out = ens.Solution(u=pg.out(), retcode=torch.empty(sh.n_local, dtype=torch.int32, device=dev),
                       n_accept=torch.empty(sh.n_local, dtype=torch.int32, device=dev),
                       n_reject=torch.empty(sh.n_local, dtype=torch.int32, device=dev), stats=None)
    for adaptive in (False, True):
        ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa, out=out, adaptive=adaptive, abstol=1e-7,
                  reltol=1e-7)
        full = pg.complete()
        if rank == 0:
            U0, P = ens.generate_inputs("lorenz", "random10", N_total, dtype=dt, seed=0xC5, N_total=N_total)
            ref = ens.solve("lorenz", "tsit5", U0, P, (0.0, 1.0), 1e-3, saveat=sa, adaptive=adaptive, abstol=1e-7,
                            reltol=1e-7)
            torch.cuda.synchronize()
            assert torch.equal(full, ref.u), (dt, adaptive)
        dist.barrier()
print("PEER_GATHER_OK", rank)
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_peer_gather_two_processes_one_gpu():
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"PEER_GATHER_OK {r}" in o, o[-3000:]


def test_out_ld_slice_equals_contiguous():
    """A solve written into a column slice of a wider array (out_ld) equals the plain solve."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 1234
    u0, p = ens.generate_inputs("lorenz", "random10", N, dtype=torch.float32, seed=3)
    big = torch.full((2, 3, 3000), float("nan"), dtype=torch.float32, device="cuda")
    sl = big[..., 777:777 + N]
    out = ens.Solution(u=sl, retcode=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_accept=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_reject=torch.empty(N, dtype=torch.int32, device="cuda"), stats=None)
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=[0.5, 1.0], out=out)
    ref = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=[0.5, 1.0])
    assert torch.equal(sl, ref.u)
    assert torch.isnan(big[..., :777]).all() and torch.isnan(big[..., 777 + N:]).all()


def test_stats_on_row_strided_slice():
    """ens_ensemble_stats with ld > N (a slice of a wider array) equals the dense computation."""
    import torch

    import paper_2304_06835_b200 as ens
    big = torch.randn((2, 3, 10000), dtype=torch.float64, device="cuda")
    sl = big[..., 1234:1234 + 7000]
    a = ens.ensemble_stats(sl)
    b = ens.ensemble_stats(sl.contiguous())
    assert torch.equal(a, b)


@pytest.mark.parametrize("model,alg,kw", [("gbm", "em", dict(seed=3)), ("robertson", "rodas5", dict(adaptive=True)),
                                          ("lorenz", "vern9", dict(adaptive=True))])
def test_out_ld_all_kernel_families(model, alg, kw):
    """out_ld on the SDE, Rosenbrock and Verner kernels (stats on for EM: the fused partials
    read the states in registers, the slice only receives them)."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 1000
    u0, p = ens.generate_inputs(model, "random10", N, dtype=torch.float64, seed=8)
    n = u0.shape[0]
    big = torch.full((2, n, 2500), float("nan"), dtype=torch.float64, device="cuda")
    sl = big[..., 300:300 + N]
    sa = [0.0, 0.5] if alg == "em" else [0.5, 1.0]
    out = ens.Solution(u=sl, retcode=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_accept=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_reject=torch.empty(N, dtype=torch.int32, device="cuda"),
                       stats=torch.empty((2, n, 3), dtype=torch.float64, device="cuda") if alg == "em" else None)
    ens.solve(model, alg, u0, p, (0.0, 1.0), 0.01, saveat=sa, out=out, stats=(alg == "em"), **kw)
    ref = ens.solve(model, alg, u0, p, (0.0, 1.0), 0.01, saveat=sa, stats=(alg == "em"), **kw)
    assert torch.equal(sl, ref.u)
    if alg == "em":
        assert torch.equal(out.stats, ref.stats)
    assert torch.isnan(big[..., :300]).all() and torch.isnan(big[..., 300 + N:]).all()
