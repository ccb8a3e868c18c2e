"""Multi-GPU ensemble driver (the paper's MPI run, done
intra-node over NCCL/NVLink instead).

Trajectories are independent, so the solve itself shards with no collective:
every rank generates and solves only its own shard on its own GPU (global
trajectory indices fix the inputs and the Philox counters, so every trajectory
is bit-identical for any world size). The two real exchange steps come after
the solve:
  1. ensemble statistics: all-gather of each rank's (count, mean, M2) triples,
     then a fixed rank-order Chan merge on every rank (deterministic);
  2. optional gather of final / saved states to rank 0 — either an NCCL
     gather after the solve, or fused into it (PeerGather: the solver stores
     into rank 0's array through CUDA IPC / NVLink while it runs).
Collectives go through torch.distributed (NCCL on GPUs; the same code runs on
gloo with CPU tensors for the host-side tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n_local: int          # trajectories on this rank
    index_offset: int     # global index of local trajectory 0
    chunk_len: int = 0    # block-cyclic layout (0 = contiguous)
    chunk_stride: int = 0

    def global_indices(self) -> torch.Tensor:
        i = torch.arange(self.n_local, dtype=torch.int64)
        if self.chunk_len > 0:
            return self.index_offset + (i // self.chunk_len) * self.chunk_stride + i % self.chunk_len
        return self.index_offset + i


def shard_contiguous(n_total: int, rank: int, world: int) -> Shard:
    """[r·N/R, (r+1)·N/R) — fixed-step runs, where work per trajectory is uniform."""
    lo = (n_total * rank) // world
    hi = (n_total * (rank + 1)) // world
    return Shard(rank, world, hi - lo, lo)


def shard_block_cyclic(n_total: int, rank: int, world: int, chunk: int = 1 << 16) -> Shard:
    """Chunks of `chunk` trajectories dealt round-robin — adaptive runs, where step
    counts correlate with the parameter sweep. Requires n_total % (chunk·world) == 0
    for a single-launch strided layout; otherwise falls back to contiguous."""
    if chunk <= 0 or n_total % (chunk * world) != 0:
        return shard_contiguous(n_total, rank, world)
    return Shard(rank, world, n_total // world, rank * chunk, chunk, chunk * world)


def shard_weak(n_per_rank: int, rank: int, world: int) -> Shard:
    """Weak scaling: a fixed n_per_rank on every rank, global ensemble = world × n_per_rank."""
    return Shard(rank, world, n_per_rank, rank * n_per_rank)


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo moves CUDA tensors through host memory (used only to exercise the
    multi-rank path on a single GPU; NCCL works on device tensors directly)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def allgather_stats(local: torch.Tensor, group=None) -> torch.Tensor:
    """[k, n, 3] per-rank (count, mean, M2) → [R, k, n, 3] on every rank."""
    R = dist.get_world_size(group)
    src = local.cpu() if _host_staged(local, group) else local.contiguous()
    out = torch.empty((R * src.shape[0], *src.shape[1:]), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.view(R, *local.shape).to(local.device)


def merge_stats(gathered: torch.Tensor) -> torch.Tensor:
    """Fixed rank-order Chan merge (device kernel ens_stats_merge)."""
    import paper_2304_06835_b200 as ens
    if not gathered.is_cuda:
        raise RuntimeError("merge_stats runs on the GPU (no CPU path)")
    return ens.stats_merge(gathered)


class PeerGather:
    """Gather fused into the solve (SURVEY §8e exchange 2): rank `dst` owns the
    global state array [*lead, N_total]; its CUDA IPC handle goes to every rank,
    which passes its column slice [*lead, off:off+N_r] as the solver's output
    (ens_options.out_ld = N_total). Each trajectory's final / saved states are
    then stored by the solver kernel straight into the destination GPU's memory
    (NVLink peer stores, P2P enabled lazily by the IPC mapping) while the solve
    runs — no separate gather collective after it. `complete()` orders the
    destination's later reads after every rank's solve: a one-element NCCL
    all-reduce on the stream (device-side), or a host barrier on gloo.

    Shards must be contiguous (`shard_contiguous` / `shard_weak`)."""

    def __init__(self, lead: tuple, n_local: int, index_offset: int, n_total: int, dtype, device, dst: int = 0,
                 group=None):
        from torch.multiprocessing.reductions import reduce_tensor
        self.group, self.dst, self.device = group, dst, torch.device(device)
        me = dist.get_rank(group)
        self.buf = None
        payload = [None]
        if me == dst:
            self.buf = torch.empty((*lead, n_total), dtype=dtype, device=self.device)
            payload = [reduce_tensor(self.buf)]
        dist.broadcast_object_list(payload, src=dst, group=group)
        if me == dst:
            remote = self.buf
        else:
            fn, args = payload[0]
            remote = fn(*args)                      # the destination's array, mapped through CUDA IPC
            if remote.device != self.device and not torch.cuda.can_device_access_peer(self.device, remote.device):
                raise RuntimeError(f"no peer access {self.device} -> {remote.device}")
        self.view = remote[..., index_offset:index_offset + n_local]
        self._flag = torch.zeros(1, dtype=torch.float32, device=self.device)

    def out(self) -> torch.Tensor:
        """This rank's slice of the destination array: pass as the solver output (Solution.u)."""
        return self.view

    def complete(self) -> Optional[torch.Tensor]:
        """After the solve: every rank's stores are ordered before the destination's reads.
        Returns the full array on `dst`, None elsewhere."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)
        return self.buf


def gather_states(local: torch.Tensor, dst: int = 0, group=None) -> Optional[torch.Tensor]:
    """Gather each rank's [..., N_r] state block to `dst` (equal N_r on all ranks).
    Returns [R, ..., N_r] on dst, None elsewhere."""
    R = dist.get_world_size(group)
    me = dist.get_rank(group)
    src = local.cpu() if _host_staged(local, group) else local.contiguous()
    if me == dst:
        bufs = [torch.empty_like(src) for _ in range(R)]
        dist.gather(src, gather_list=bufs, dst=dst, group=group)
        return torch.stack(bufs).to(local.device)
    dist.gather(src, dst=dst, group=group)
    return None


@dataclass
class MultiSolution:
    """Result of `solve` on one rank."""
    shard: Shard
    local: "object"                      # this rank's ens.Solution (u may be a view into dst's gather array)
    stats: Optional[torch.Tensor]        # merged [max(k,1), n, 3] (count, mean, M2) on every rank, or None
    gathered: Optional[torch.Tensor]     # on dst: [*lead, N_total] in global order (gather="peer"), or
    #                                      [R, *lead, N_r] rank blocks (gather="nccl"); None elsewhere / no gather


def solve(model: str, alg: str, recipe: str, N_total: int, tspan, dt, *, dtype=torch.float32, input_seed: int = 0,
          shard: str = "auto", chunk: int = 1 << 16, gather: Optional[str] = None, dst: int = 0, stats: bool = False,
          saveat=None, group=None, device=None, **solve_kw) -> MultiSolution:
    """The multi-rank driver (SURVEY §8b `ens.multi_gpu.solve`, §8e): call on every rank of an
    initialised process group, one rank per GPU.

    1. shard the N_total trajectories: "contiguous", "block_cyclic" (chunks of `chunk` dealt round-robin,
       one launch per rank through ens_options.chunk_len / chunk_stride), or "auto" (block-cyclic for
       adaptive runs when N_total divides evenly and gather != "peer", contiguous otherwise);
    2. generate this shard's inputs on the rank's GPU from (input_seed, global index) — no scatter;
    3. solve the shard (global indices key the Philox noise, so every trajectory is bit-identical for
       any world size);
    4. stats=True: per-rank (count, mean, M2) — fused in the EM kernels and the fixed-step Tsit5
       epilogue, a reduction pass over the stored states otherwise — all-gathered and merged in
       fixed rank order on every rank;
    5. gather="peer": the solver stores straight into dst's [*lead, N_total] array (PeerGather; contiguous
       shards only); gather="nccl": NCCL gather of the rank blocks after the solve (equal N_r).
    `solve_kw` goes to ens.solve (adaptive, abstol, reltol, seed, refill, max_steps, ...)."""
    import paper_2304_06835_b200 as ens
    R, me = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    adaptive = bool(solve_kw.get("adaptive", False))
    if shard == "auto":
        # peer gather needs contiguous shards (each rank writes one column slice of dst's array)
        shard = "block_cyclic" if adaptive and gather != "peer" and N_total % (chunk * R) == 0 else "contiguous"
    if shard == "block_cyclic":
        if gather == "peer":
            raise ValueError("gather='peer' needs contiguous shards")
        sh = shard_block_cyclic(N_total, me, R, chunk)
    elif shard == "contiguous":
        sh = shard_contiguous(N_total, me, R)
    else:
        raise ValueError(f"unknown shard layout {shard!r}")
    if gather == "nccl" and N_total % R != 0:
        raise ValueError("gather='nccl' needs equal shards (N_total divisible by the world size)")
    if gather not in (None, "peer", "nccl"):
        raise ValueError(f"unknown gather {gather!r}")

    u0, p = ens.generate_inputs(model, recipe, sh.n_local, dtype=dtype, seed=input_seed, index_offset=sh.index_offset,
                                N_total=N_total, chunk_len=sh.chunk_len, chunk_stride=sh.chunk_stride, device=dev)
    n, _, _ = ens.model_dims(model)
    k = 0 if saveat is None else len(saveat)
    lead = (k, n) if k else (n,)
    sde = alg in ("em", "siea")
    pg = PeerGather(lead, sh.n_local, sh.index_offset, N_total, dtype, dev, dst=dst, group=group) \
        if gather == "peer" else None
    out = None
    if pg is not None:
        out = ens.Solution(u=pg.out(), retcode=torch.empty(sh.n_local, dtype=torch.int32, device=dev),
                           n_accept=torch.empty(sh.n_local, dtype=torch.int32, device=dev),
                           n_reject=torch.empty(sh.n_local, dtype=torch.int32, device=dev),
                           stats=torch.empty((max(k, 1), n, 3), dtype=torch.float64, device=dev)
                           if stats else None)
    # statistics come from the solve: fused into the EM kernels and the fixed-step Tsit5 epilogue,
    # else a pass over the stored states run on this rank's GPU
    sol = ens.solve(model, alg, u0, p, tspan, dt, saveat=saveat, stats=stats, out=out,
                    store_states=(gather is not None) or not (stats and sde),
                    index_offset=sh.index_offset, chunk_len=sh.chunk_len, chunk_stride=sh.chunk_stride, **solve_kw)
    merged = merge_stats(allgather_stats(sol.stats, group)) if stats else None
    gathered = None
    if pg is not None:
        gathered = pg.complete()
    elif gather == "nccl":
        gathered = gather_states(sol.u, dst=dst, group=group)
    return MultiSolution(sh, sol, merged, gathered)
