"""Multi-GPU ensemble driver (the paper's MPI run, done
intra-node over NCCL/NVLink instead).

Trajectories are independent, so the solve itself shards with no collective:
every rank generates and solves only its own shard on its own GPU (global
trajectory indices fix the inputs and the Philox counters, so every trajectory
is bit-identical for any world size). The two real exchange steps come after
the solve:
  1. ensemble statistics: all-gather of each rank's (count, mean, M2) triples,
     then a fixed rank-order Chan merge on every rank (deterministic);
  2. optional gather of final / saved states to rank 0.
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
