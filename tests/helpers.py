"""Shared test helpers (no method arithmetic): run both sides on the same seeded inputs."""
from __future__ import annotations

import json
import os

import numpy as np

NP = {"f32": np.float32, "f64": np.float64}


def traj_relerr(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per-trajectory norm-wise relative error: max over (points, components) of
    |got − ref| / max(|ref|) (∞-norm of the trajectory's values; arrays are
    [..., N] with the trajectory index last)."""
    g = got.reshape(-1, got.shape[-1]).astype(np.float64)
    r = ref.reshape(-1, ref.shape[-1]).astype(np.float64)
    both_nan = np.isnan(g) & np.isnan(r)          # unreached save points (DESIGN R6) agree
    d = np.where(both_nan, 0.0, np.abs(g - r))
    scale = np.maximum(np.nanmax(np.where(np.isnan(r), 0.0, np.abs(r)), axis=0), np.finfo(np.float64).tiny)
    return d.max(0) / scale


def bitexact(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per trajectory: every stored value identical (NaN == NaN)."""
    g = got.reshape(-1, got.shape[-1])
    r = ref.reshape(-1, ref.shape[-1]).astype(g.dtype)
    return ((g == r) | (np.isnan(g) & np.isnan(r))).all(0)


def parity_log(name: str | None, **rec) -> dict:
    """Print a parity record and append it (JSON line) to $PARITY_LOG if set, so the
    measured match rates of a GPU run can be committed (profiles/parity_rates_*.jsonl).
    name=None: the running pytest test id (with parameters)."""
    if name is None:
        name = os.environ.get("PYTEST_CURRENT_TEST", "?").rsplit(" (", 1)[0]
    rec = {"test": name, **{k: (float(v) if isinstance(v, (np.floating, np.integer)) else v) for k, v in rec.items()}}
    print("PARITY " + json.dumps(rec))
    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


def check_fixed(g, o, tol: float, *, name: str | None = None, bitexact_min: float = 0.99):
    """Fixed-step parity (north star: rel ≤ 1e-12 fp64 / 1e-5 fp32 on every
    trajectory); canonical operation order on both sides makes most
    trajectories bit-exact, which is checked too."""
    rel = traj_relerr(g, o)
    be = bitexact(g, o)
    parity_log(name, n=int(rel.size), bitexact_frac=be.mean(), max_rel=rel.max())
    assert rel.max() <= tol, (name, rel.max())
    assert be.mean() >= bitexact_min, (name, be.mean())


def check_adaptive(g, o, counts_g, counts_o, *, tol: float, name: str | None = None, same_min: float = 0.999,
                   ref=None, tol_same: float | None = None):
    """Adaptive parity on EVERY trajectory.

    counts_g / counts_o: (n_accept,) or (n_accept, n_reject) arrays of each side.
    Identical step counts on ≥ same_min of the trajectories (north star 99.9 %).
    fp64 (ref is None): final / saved states within `tol` on all trajectories.
    fp32 (ref = a tight fp64 reference solution of the same inputs): trajectories
    with identical counts agree within `tol_same` (rounding level); any whose step
    sequence differs must still be as accurate as the oracle's own fp32 solutions —
    GPU error against ref ≤ 2 × the oracle's largest error against ref (in fp32 at
    these tolerances a one-ulp difference re-routes the step sequence, DESIGN R2),
    and all trajectories within `tol`."""
    same = np.ones(np.shape(counts_g[0]), bool)
    for a, b in zip(counts_g, counts_o):
        same &= np.asarray(a) == np.asarray(b)
    rel = traj_relerr(g, o)
    be = bitexact(g, o)
    rec = dict(n=int(rel.size), same_counts=same.mean(), bitexact_frac=be.mean(), max_rel=rel.max(),
               max_rel_same=rel[same].max() if same.any() else 0.0,
               max_rel_mismatched=rel[~same].max() if (~same).any() else 0.0)
    if ref is not None:
        eo = traj_relerr(o, ref)
        eg = traj_relerr(g, ref)
        rec.update(oracle_err_vs_ref=eo.max(), gpu_err_vs_ref=eg.max())
    parity_log(name, **rec)
    assert same.mean() >= same_min, (name, same.mean())
    assert rel.max() <= tol, (name, rel.max())
    if tol_same is not None and same.any():
        assert rel[same].max() <= tol_same, (name, rel[same].max())
    if ref is not None and (~same).any():
        assert eg[~same].max() <= 2.0 * eo.max(), (name, eg[~same].max(), eo.max())


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
