"""torchrun worker for tests/test_multi_gpu_nccl.py (one rank per GPU, NCCL).

Each rank generates and solves only its shard (global indices), computes the
shard's statistics, all-gathers and merges them, and gathers its final states
to rank 0. Rank 0 checks against one single-process solve of the whole
ensemble: states bit-identical (partition independence), merged statistics
within 1e-13 relative."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2304_06835_b200 as ens  # noqa: E402
from paper_2304_06835_b200 import multi_gpu as mg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    N_total = 40960 * world
    for mode in ["fixed", "adaptive"]:
        maker = mg.shard_contiguous if mode == "fixed" else (lambda n, r, w: mg.shard_block_cyclic(n, r, w, 4096))
        sh = maker(N_total, rank, world)
        u0, p = ens.generate_inputs("lorenz", "random10", sh.n_local, dtype=torch.float32, seed=0xC5,
                                    index_offset=sh.index_offset, chunk_len=sh.chunk_len,
                                    chunk_stride=sh.chunk_stride, device=dev)
        kw = dict(adaptive=True, abstol=1e-6, reltol=1e-6, refill=True) if mode == "adaptive" else {}
        sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, **kw)
        st = ens.ensemble_stats(sol.u.view(1, 3, -1))
        merged = mg.merge_stats(mg.allgather_stats(st))
        g = mg.gather_states(sol.u)
        if rank == 0:
            U0, P = ens.generate_inputs("lorenz", "random10", N_total, dtype=torch.float32, seed=0xC5, device=dev)
            ref = ens.solve("lorenz", "tsit5", U0, P, (0.0, 1.0), 1e-3, **kw)
            ref_st = ens.ensemble_stats(ref.u.view(1, 3, -1))
            for r in range(world):
                shr = maker(N_total, r, world)
                gi = shr.global_indices().to(dev)
                assert torch.equal(g[r], ref.u[:, gi]), (mode, r)
            rel = ((merged[..., 1] - ref_st[..., 1]).abs() / ref_st[..., 1].abs()).max().item()
            relv = ((merged[..., 2] - ref_st[..., 2]).abs() / ref_st[..., 2].abs()).max().item()
            assert merged[..., 0].eq(N_total).all().item()
            assert rel <= 1e-13 and relv <= 1e-12, (mode, rel, relv)
    dist.barrier()
    if rank == 0:
        print("MGPU_OK", world, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
