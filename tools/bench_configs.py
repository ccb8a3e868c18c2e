#!/usr/bin/env python
"""Time every BASELINE.json config at full size on one GPU.

Prints one JSON line per (config, variant): trajectories/s, kernel ms (CUDA
events, best of R after warm-up, "taking the best timing"), attempted
steps, achieved FLOP/s vs the FP peak (fixed / adaptive Tsit5, Rosenbrock23),
HBM GB/s for saveat-heavy runs. Inputs are generated on device; no oracle here
(parity lives in tests/).
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2304_06835_b200 as ens  # noqa: E402

SMS = 148
PEAK = {"f32": SMS * 128 * 2 * 1965e6, "f64": SMS * 64 * 2 * 1965e6}
HBM = 6536.7e9
T = {"f32": torch.float32, "f64": torch.float64}
# algorithmic FLOPs per attempted step
FLOP_STEP = {"tsit5_fixed": 192.0, "tsit5_adaptive": 265.0, "ros23": 170.0}


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


ONLY: list[str] = []


def run(name, model, alg, recipe, N, dtype, tspan, dt, flop_key=None, reps=5, **kw):
    if ONLY and not any(name.startswith(o) for o in ONLY):
        return None
    u0, p = ens.generate_inputs(model, recipe, N, dtype=T[dtype], seed=kw.pop("input_seed", 0), N_total=N)
    if kw.pop("shuffle", False):
        perm = torch.randperm(N, generator=torch.Generator().manual_seed(1)).cuda()
        u0, p = u0[:, perm].contiguous(), (p[:, perm].contiguous() if p.dim() == 2 else p)
    sa = kw.get("saveat")
    k = 0 if sa is None else len(sa)
    n = u0.shape[0]
    out = ens.Solution(u=torch.empty((k, n, N) if k else (n, N), dtype=T[dtype], device="cuda")
                       if kw.get("store_states", True) else None,
                       retcode=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_accept=torch.empty(N, dtype=torch.int32, device="cuda"),
                       n_reject=torch.empty(N, dtype=torch.int32, device="cuda"),
                       stats=torch.empty((max(k, 1), n, 3), dtype=torch.float64, device="cuda")
                       if kw.get("stats") else None)
    ws = ens.Workspace(1 << 20, "cuda")
    kw.pop("store_states", None)
    ms = timeit(lambda: ens.solve(model, alg, u0, p, tspan, dt, out=out, workspace=ws, **kw), reps=reps)
    na = out.n_accept.to(torch.int64)
    nr = out.n_reject.to(torch.int64)
    att = int((na + nr).sum().item())
    ok = float((out.retcode == 0).float().mean().item())
    line = {"config": name, "model": model, "alg": alg, "N": N, "dtype": dtype, "ms": ms,
            "traj_per_s": N / (ms / 1e3), "success_frac": ok,
            "steps_mean": att / N, "steps_min": int((na + nr).min().item()), "steps_max": int((na + nr).max().item()),
            "opts": {k2: (v if not isinstance(v, (list, tuple)) or len(v) < 5 else f"{len(v)} points")
                     for k2, v in kw.items()}}
    if flop_key:
        fl = att * FLOP_STEP[flop_key]
        line["achieved_tflops"] = fl / (ms / 1e3) / 1e12
        line["frac_fp_peak"] = fl / (ms / 1e3) / PEAK[dtype]
    if k:
        bytes_out = k * n * N * (4 if dtype == "f32" else 8)
        line["saveat_GBps"] = bytes_out / (ms / 1e3) / 1e9
        line["saveat_frac_hbm"] = bytes_out / (ms / 1e3) / HBM
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="", help="comma-separated config-name prefixes")
    args = ap.parse_args()
    ONLY[:] = [o for o in args.only.split(",") if o]
    big = 10**6 if args.quick else 10**7
    # C1: Lorenz N=1024, random p ±10 %, fp64 adaptive 1e-8 (latency regime)
    for refill in [False, True]:
        run("C1", "lorenz", "tsit5", "random10", 1024, "f64", (0.0, 1.0), 1e-3, "tsit5_adaptive", reps=20,
            input_seed=0xC1, adaptive=True, abstol=1e-8, reltol=1e-8, refill=refill)
    # NEXT-1: C1 on Vern7, and Tsit5 vs Vern7 at the north_star's tight fp64 tolerance (1e-10)
    for alg in ["vern7", "vern9"]:
        for refill in [False, True]:
            run("C1-" + alg, "lorenz", alg, "random10", 1024, "f64", (0.0, 1.0), 1e-3, None, reps=20,
                input_seed=0xC1, adaptive=True, abstol=1e-8, reltol=1e-8, refill=refill)
    for alg in ["tsit5", "vern7", "vern9"]:
        run("tight-" + alg, "lorenz", alg, "rho_sweep", 10**6, "f64", (0.0, 1.0), 1e-3, None, reps=3,
            adaptive=True, abstol=1e-10, reltol=1e-10, refill=True)
    run("C2-fixed-vern7", "lorenz", "vern7", "rho_sweep", big, "f32", (0.0, 1.0), 1e-3, None)
    # C2: Lorenz ρ sweep, fixed dt=1e-3 and adaptive 1e-6, fp32 (and fp64 fixed)
    for N in [10**3, 10**4, 10**5, 10**6, big]:
        run("C2-fixed", "lorenz", "tsit5", "rho_sweep", N, "f32", (0.0, 1.0), 1e-3, "tsit5_fixed")
        for refill in [False, True]:
            run("C2-adaptive", "lorenz", "tsit5", "rho_sweep", N, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive",
                adaptive=True, abstol=1e-6, reltol=1e-6, refill=refill)
    run("C2-fixed", "lorenz", "tsit5", "rho_sweep", big, "f64", (0.0, 1.0), 1e-3, "tsit5_fixed")
    # saveat-dense: every one of the 1001 grid points stored, [1001][3][N] fp32 — the HBM-write
    # side of the roofline (12 B per trajectory-step against 192 FLOP)
    sa_all = [j * 1e-3 for j in range(1001)]
    sa_all[-1] = 1.0
    for Nd in [10**6, 4 * 10**6]:
        run("C2-saveat-dense", "lorenz", "tsit5", "rho_sweep", Nd, "f32", (0.0, 1.0), 1e-3, "tsit5_fixed", reps=3,
            saveat=sa_all)
    # the C2 adaptive ensemble with its columns randomly permuted: neighbouring lanes no longer have
    # similar step counts (20-47), the divergence the refill scheduler (a8) is for
    for refill in [False, True]:
        run("C2-adaptive-shuffled", "lorenz", "tsit5", "rho_sweep", big, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive",
            adaptive=True, abstol=1e-6, reltol=1e-6, refill=refill, shuffle=True)
    # C3: Robertson N=10^6 fp64 Rosenbrock23 adaptive 1e-8, saveat 100 points (2.4 GB of states)
    sa = [1e5 * j / 99 for j in range(100)]
    for refill in [False, True]:
        run("C3", "robertson", "rosenbrock23", "random10", 10**6, "f64", (0.0, 1e5), 1e-4, "ros23", reps=3,
            input_seed=0xC3, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa, refill=refill)
    # NEXT-2: the C3 workload on Rodas4 (4th order: far fewer steps at the same tolerance)
    for refill in [False, True]:
        run("C3-rodas4", "robertson", "rodas4", "random10", 10**6, "f64", (0.0, 1e5), 1e-4, None, reps=3,
            input_seed=0xC3, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa, refill=refill)
    for refill in [False, True]:
        run("C3-rodas5", "robertson", "rodas5", "random10", 10**6, "f64", (0.0, 1e5), 1e-4, None, reps=3,
            input_seed=0xC3, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa, refill=refill)
        run("C3-rodas5p", "robertson", "rodas5p", "random10", 10**6, "f64", (0.0, 1e5), 1e-4, None, reps=3,
            input_seed=0xC3, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa, refill=refill)
    # C4: stochastic Lorenz EM dt=1e-3, 10^6 paths, 11 save points, ensemble mean/var
    sa4 = [j / 10 for j in range(11)]
    for model in ["lorenz_sde_add", "lorenz_sde_mul"]:
        for dt_ in ["f32", "f64"]:
            run("C4", model, "em", "const", 10**6, dt_, (0.0, 1.0), 1e-3, None, reps=3, seed=0xC4, saveat=sa4,
                stats=True, store_states=False)
    # NEXT-3: σ-factor CRN SDE, 10^6-point parameter grid, dt = 0.1 on [0, 1000], stats every 100
    sa6 = [100.0 * j for j in range(11)]
    for dt_ in ["f32", "f64"]:
        run("CRN", "crn", "em", "grid", 10**6 if not args.quick else 10**5, dt_, (0.0, 1000.0), 0.1, None, reps=2,
            seed=0xC7, saveat=sa6, stats=True, store_states=False)
    # NEXT-4: stiff suite at the paper's 8192 trajectories, Rosenbrock23 fp64, tol 1e-8
    for model, tf in [("orego", 30.0), ("hires", 321.8122), ("pollu", 60.0)]:
        run("stiff-" + model, model, "rosenbrock23", "random10", 8192, "f64", (0.0, tf), 1e-6, "ros23", reps=3,
            input_seed=0x57, adaptive=True, abstol=1e-8, reltol=1e-8)
        for alg in ["rodas4", "rodas5", "rodas5p"]:
            run(f"stiff-{alg}-" + model, model, alg, "random10", 8192, "f64", (0.0, tf), 1e-6, None, reps=3,
                input_seed=0x57, adaptive=True, abstol=1e-8, reltol=1e-8)
    # C5: Lorenz fp32 10^8 on one GPU (the 8-GPU run shards this), random p ±10 %
    if not args.quick:
        run("C5-1gpu", "lorenz", "tsit5", "random10", 10**8, "f32", (0.0, 1.0), 1e-3, "tsit5_fixed", reps=2,
            input_seed=0xC5)
        run("C5-1gpu-adaptive", "lorenz", "tsit5", "random10", 10**8, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive",
            reps=2, input_seed=0xC5, adaptive=True, abstol=1e-6, reltol=1e-6, refill=True)


if __name__ == "__main__":
    main()
