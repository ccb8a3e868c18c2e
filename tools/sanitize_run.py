#!/usr/bin/env python
"""Small solves touching every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2304_06835_b200 as ens  # noqa: E402

dev = torch.device("cuda:0")
N = 333   # ragged: several blocks + a tail; odd → a dead partner lane in the fp32 pair kernel
for dt in [torch.float32, torch.float64]:
    u0, p = ens.generate_inputs("lorenz", "random10", N, dtype=dt, seed=1)
    sa = np.linspace(0, 1, 5)
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2)
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2, stats=True)          # fused statistics (fixed step)
    ul, pl = ens.generate_inputs("lorenz", "random10", 600_001, dtype=dt, seed=2)  # > 8192 partials: fold + merge
    ens.solve("lorenz", "tsit5", ul, pl, (0.0, 1.0), 0.25, stats=True)
    del ul, pl
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2, saveat=sa, stats=True)
    ub2, pb2 = ens.generate_inputs("lorenz", "random10", 1100, dtype=dt, seed=6)   # full blocks + a tail
    ens.solve("lorenz", "tsit5", ub2, pb2, (0.0, 1.0), 1e-2, saveat=np.arange(0, 101) * 1e-2)   # grid saves
    ens.solve("lorenz", "tsit5", ub2, pb2, (0.0, 1.0), 1e-2, saveat=np.arange(0, 101) * 1e-2,
              bulk_saves=True)                                                                  # cp.async.bulk path
    ens.solve("lorenz", "tsit5", ub2, pb2, (0.0, 1.0), 1e-2, saveat=[0.0, 0.333, 1.0])      # interpolated
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6)
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6,
              saveat=[0.0, 0.123, 0.5, 1.0])                        # static (fp32: component-pair kernel) + saves
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6, refill=True,
              saveat=sa)
    ur, pr = ens.generate_inputs("robertson", "random10", N, dtype=dt, seed=3)
    ens.solve("robertson", "rosenbrock23", ur, pr, (0.0, 10.0), 1e-4, adaptive=True, abstol=1e-6, reltol=1e-6,
              saveat=np.linspace(0, 10, 4))
    ens.solve("robertson", "rosenbrock23", ur, pr, (0.0, 10.0), 1e-4, adaptive=True, abstol=1e-6, reltol=1e-6,
              refill=True)
    # Lorenz W = I − h d J needs row exchanges in some warps: the LU fast path's vote + rebuild
    ens.solve("lorenz", "rosenbrock23", u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6)
    ens.solve("lorenz", "rodas5", u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6)
    for alg in ["rodas4", "rodas5", "rodas5p"]:
        ens.solve("robertson", alg, ur, pr, (0.0, 10.0), 1e-4, adaptive=True, abstol=1e-6, reltol=1e-6,
                  saveat=np.linspace(0, 10, 4))
        ens.solve("robertson", alg, ur, pr, (0.0, 10.0), 1e-4, adaptive=True, abstol=1e-6, reltol=1e-6, refill=True)
        ens.solve("robertson", alg, ur, pr, (0.0, 1.0), 0.01, saveat=[0.0, 0.5, 1.0])
        ens.solve("robertson", alg, ur, pr, (0.0, 1.0), 0.01, saveat=[0.0, 0.257, 0.5, 0.9999])   # off-grid (R24)
    for alg in ["vern7", "vern9"]:
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6, saveat=sa)
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, adaptive=True, abstol=1e-6, reltol=1e-6, refill=True)
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, saveat=[0.0, 0.5, 1.0])
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, saveat=[0.0, 0.005, 0.5, 0.777, 1.0])   # off-grid (R24)
    us, ps = ens.generate_inputs("lorenz_sde_mul", "const", N, dtype=dt)
    ens.solve("lorenz_sde_mul", "em", us, ps, (0.0, 0.1), 1e-3, seed=5, saveat=np.linspace(0, 0.1, 3), stats=True,
              store_states=False)
    uc, pc = ens.generate_inputs("crn", "grid", N, dtype=dt, N_total=10**6)
    ens.solve("crn", "em", uc, pc, (0.0, 1.0), 0.1, seed=7, stats=True)
    ub, pb = ens.generate_inputs("ball", "random10", N, dtype=dt, seed=2)
    ens.solve("ball", "tsit5", ub, pb, (0.0, 15.0), 0.1, adaptive=True, abstol=1e-6, reltol=1e-6)
    ens.sde_noise(N, 2, seed=1, dtype=dt, nw=8)
    x = torch.randn((2, 3, N), dtype=dt, device=dev)
    st = ens.ensemble_stats(x)
    ens.stats_finalize(st)
    ens.stats_merge(torch.stack([st, st]))
uh, ph = ens.generate_inputs("hires", "random10", 64, dtype=torch.float64, seed=4)
ens.solve("hires", "rosenbrock23", uh, ph, (0.0, 5.0), 1e-6, adaptive=True, abstol=1e-6, reltol=1e-6)
up, pp = ens.generate_inputs("pollu", "random10", 40, dtype=torch.float64, seed=4)
ens.solve("pollu", "rosenbrock23", up, pp, (0.0, 1.0), 1e-6, adaptive=True, abstol=1e-6, reltol=1e-6)
ens.solve("pollu", "rodas5", up, pp, (0.0, 1.0), 1e-6, adaptive=True, abstol=1e-6, reltol=1e-6)
ens.solve("hires", "rodas4", uh, ph, (0.0, 5.0), 1e-6, adaptive=True, abstol=1e-6, reltol=1e-6, saveat=[1.0, 2.0])
u0h, p0h = (t.cpu().pin_memory() for t in ens.generate_inputs("lorenz", "random10", N, dtype=torch.float32))
ens.solve_host("lorenz", "tsit5", u0h, p0h, (0.0, 1.0), 1e-2, n_chunks=3)
ush, psh = (t.cpu().pin_memory() for t in ens.generate_inputs("gbm", "random10", N, dtype=torch.float64))
ens.solve_host("gbm", "em", ush, psh, (0.0, 1.0), 1e-2, n_chunks=3, seed=3, index_offset=100)
torch.cuda.synchronize()
print("SANITIZE_RUN_OK")
