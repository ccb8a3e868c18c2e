#!/usr/bin/env python
"""Run one config a few times (for ncu capture). Usage: prof_one.py NAME [N]
NAME: c2f32 / c2f64 (Lorenz tsit5 fixed, rho sweep, fused stats), c1t (Lorenz tsit5 fp64 1e-10 rho sweep),
c2a (Lorenz tsit5 adaptive fp32 1e-6 rho sweep), c3 (Robertson ros23 fp64
saveat 100), c3r5 (the same on Rodas5), c4 (stochastic Lorenz EM fp32 stats),
c4d (the same fp64), c1 (Lorenz fp64 adaptive 1e-8), tight9 / tight7 (Lorenz fp64
1e-10 on Vern9 / Vern7, refill), t9 / t7 (the same, static mapping)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2304_06835_b200 as ens

args = [x for x in sys.argv[1:] if not x.startswith("--lib=")]
for x in sys.argv[1:]:
    if x.startswith("--lib="):        # an experimental variant (tools/build_variant.py)
        ens._LIB_PATH = Path(x.split("=", 1)[1]).resolve()
name = args[0]
N = int(args[1]) if len(args) > 1 else None
reps = 3
if name == "c2a":
    N = N or 10**7
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6)
elif name in ("c2a_refill", "c2a_shuf", "c2a_shuf_refill"):
    N = N or 10**7
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    if "shuf" in name:
        perm = torch.randperm(N, generator=torch.Generator().manual_seed(1)).cuda()
        u0, p = u0[:, perm].contiguous(), p[:, perm].contiguous()
    rf = name.endswith("refill")
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6,
                          refill=rf)
elif name in ("c2f32", "c2f64"):
    N = N or 10**7
    dt_ = torch.float32 if name == "c2f32" else torch.float64
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=dt_, N_total=N)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, stats=True)
elif name == "c1t":
    N = N or 10**6
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float64, N_total=N)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10)
elif name == "dense":
    N = N or 10**6
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    sa = [j * 1e-3 for j in range(1001)]
    sa[-1] = 1.0
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
elif name == "c1":
    N = N or 1024
    u0, p = ens.generate_inputs("lorenz", "random10", N, dtype=torch.float64, seed=0xC1)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-8, reltol=1e-8)
elif name == "c3":
    N = N or 10**6
    u0, p = ens.generate_inputs("robertson", "random10", N, dtype=torch.float64, seed=0xC3)
    sa = [1e5 * j / 99 for j in range(100)]
    f = lambda: ens.solve("robertson", "rosenbrock23", u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                          reltol=1e-8, saveat=sa)
elif name in ("c3r5", "c3r5p"):
    N = N or 10**6
    u0, p = ens.generate_inputs("robertson", "random10", N, dtype=torch.float64, seed=0xC3)
    sa = [1e5 * j / 99 for j in range(100)]
    alg = "rodas5" if name == "c3r5" else "rodas5p"
    f = lambda: ens.solve("robertson", alg, u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                          reltol=1e-8, saveat=sa)
elif name in ("tight9", "tight7", "t9", "t7"):
    N = N or 10**6
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float64, N_total=N)
    alg = "vern9" if name.endswith("9") else "vern7"
    rf = name.startswith("tight")     # tight*: refill scheduler; t9 / t7: static, as bench.py's side measurement
    f = lambda: ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10,
                          refill=rf)
elif name == "c4d":
    N = N or 10**6
    u0, p = ens.generate_inputs("lorenz_sde_add", "const", N, dtype=torch.float64)
    sa = [j / 10 for j in range(11)]
    f = lambda: ens.solve("lorenz_sde_add", "em", u0, p, (0.0, 1.0), 1e-3, seed=0xC4, saveat=sa, stats=True,
                          store_states=False)
elif name == "c4":
    N = N or 10**6
    u0, p = ens.generate_inputs("lorenz_sde_add", "const", N, dtype=torch.float32)
    sa = [j / 10 for j in range(11)]
    f = lambda: ens.solve("lorenz_sde_add", "em", u0, p, (0.0, 1.0), 1e-3, seed=0xC4, saveat=sa, stats=True,
                          store_states=False)
for _ in range(reps):
    f()
torch.cuda.synchronize()
print("ok", name, N)
