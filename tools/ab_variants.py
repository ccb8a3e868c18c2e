#!/usr/bin/env python
"""A/B timing of libens.so variants (tools/build_variant.py) on one GPU.

  python tools/ab_variants.py CONFIG[,CONFIG...] VARIANT [VARIANT ...]   (VARIANT "base" = the product library)

Each (variant, config) runs in a fresh process with the binding pointed at that
variant's library; prints one JSON line with the best-of-R kernel time (CUDA
events) and a checksum of the outputs (bit-identity across variants is checked by
comparing the checksums). Configs: c3 (Robertson Rosenbrock23 fp64 1e-8, saveat
100, N=10^6), c3r5 / c3r4 (the same on Rodas5 / Rodas4), c2a (Lorenz Tsit5 fp32 1e-6 ρ sweep,
N=10^7), c1t (Lorenz Tsit5 fp64 1e-10 ρ sweep, N=10^6), t9 / t7 (the same on Vern9 / Vern7),
c2f (Lorenz Tsit5 fixed fp32 10^7), dense / dense1 (the same with all 1001 grid points saved, N = 4·10^6 / 10^6), orego/hires/pollu (stiff suite, Rosenbrock23, 8192; suffix 4 / 5:
Rodas4 / Rodas5; suffix 5p: Rodas5P; AB_REFILL=1 in the environment: the refill scheduler)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import sys, json, hashlib
sys.path.insert(0, ".")
import torch
import paper_2304_06835_b200 as ens
from pathlib import Path
var, cfg = sys.argv[1], sys.argv[2]
if var != "base":
    ens._LIB_PATH = Path("paper_2304_06835_b200/_variants") / var / "libens.so"
F64, F32 = torch.float64, torch.float32
if cfg in ("c3", "c3r5", "c3r4", "c3r5p"):
    u0, p = ens.generate_inputs("robertson", "random10", 10**6, dtype=F64, seed=0xC3)
    sa = [1e5 * j / 99 for j in range(100)]
    alg = {"c3": "rosenbrock23", "c3r5": "rodas5", "c3r4": "rodas4", "c3r5p": "rodas5p"}[cfg]
    f = lambda: ens.solve("robertson", alg, u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
elif cfg == "c2a":
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", 10**7, dtype=F32, N_total=10**7)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6)
elif cfg in ("c1t", "t9", "t7"):
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", 10**6, dtype=F64, N_total=10**6)
    alg = {"c1t": "tsit5", "t9": "vern9", "t7": "vern7"}[cfg]
    f = lambda: ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10)
elif cfg in ("dense", "dense1"):
    N = 4 * 10**6 if cfg == "dense" else 10**6
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=F32, N_total=N)
    sa = [j * 1e-3 for j in range(1001)]
    sa[-1] = 1.0
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
elif cfg == "c2f":
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", 10**7, dtype=F32, N_total=10**7)
    f = lambda: ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, stats=True)
elif cfg.rstrip("45p") in ("orego", "hires", "pollu"):
    mdl = cfg.rstrip("45p")
    alg = "rodas5p" if cfg.endswith("5p") else {"4": "rodas4", "5": "rodas5"}.get(cfg[-1], "rosenbrock23")
    tf = {"orego": 30.0, "hires": 321.8122, "pollu": 60.0}[mdl]
    u0, p = ens.generate_inputs(mdl, "random10", 8192, dtype=F64, seed=0x57)
    import os
    rf = os.environ.get("AB_REFILL", "0") == "1"
    f = lambda: ens.solve(mdl, alg, u0, p, (0.0, tf), 1e-6, adaptive=True, abstol=1e-8, reltol=1e-8, refill=rf)
sol = f(); torch.cuda.synchronize()
best = 1e30
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sol = f(); b.record(); torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
h = hashlib.sha1(sol.u.cpu().numpy().tobytes() + sol.n_accept.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps({"variant": var, "config": cfg, "ms": best, "checksum": h}))
'''


def main():
    cfgs = sys.argv[1].split(",")
    for cfg in cfgs:
        for var in sys.argv[2:]:
            r = subprocess.run([sys.executable, "-c", CHILD, var, cfg], cwd=ROOT, capture_output=True, text=True,
                               timeout=900)
            out = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            print(out[-1] if out else json.dumps({"variant": var, "config": cfg, "error": r.stderr[-500:]}),
                  flush=True)


if __name__ == "__main__":
    main()
