"""Shared test helpers (no method arithmetic): run both sides on the same seeded inputs."""
from __future__ import annotations

import numpy as np

NP = {"f32": np.float32, "f64": np.float64}


def traj_relerr(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per-trajectory norm-wise relative error: max over (points, components) of
    |got − ref| / max(|ref|) (∞-norm of the trajectory's values; arrays are
    [..., N] with the trajectory index last)."""
    g = got.reshape(-1, got.shape[-1]).astype(np.float64)
    r = ref.reshape(-1, ref.shape[-1]).astype(np.float64)
    scale = np.maximum(np.abs(r).max(0), np.finfo(np.float64).tiny)
    return np.abs(g - r).max(0) / scale


def gpu(model, alg, u0, p, tspan, dt, **kw):
    """Run the CUDA path through the C ABI on numpy inputs; returns numpy outputs."""
    import torch

    import paper_2304_06835_b200 as ens
    dev = torch.device("cuda:0")
    sol = ens.solve(model, alg, torch.from_numpy(np.ascontiguousarray(u0)).to(dev),
                    torch.from_numpy(np.ascontiguousarray(p)).to(dev), tspan, dt, **kw)
    torch.cuda.synchronize()
    u = None if sol.u is None else sol.u.cpu().numpy()
    if u is not None and u.ndim == 2:
        u = u[None]
    st = None if sol.stats is None else sol.stats.cpu().numpy()
    return u, sol.retcode.cpu().numpy(), sol.n_accept.cpu().numpy(), sol.n_reject.cpu().numpy(), st


def sample_indices(N: int, head: int = 2048, tail: int = 2048, stride_count: int = 4096, seed: int = 0):
    """Deterministic index subsample for full-size parity: first/last blocks + a spread sample."""
    idx = set(range(min(head, N))) | set(range(max(0, N - tail), N))
    rng = np.random.default_rng(seed)
    idx |= set(rng.choice(N, size=min(stride_count, N), replace=False).tolist())
    return np.array(sorted(idx), dtype=np.int64)
