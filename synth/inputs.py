"""Seeded synthetic ensemble inputs — the ONE module both sides may use.

Holds none of the method's arithmetic: only the input recipe (DESIGN.md §6,
SURVEY.md 8c.6) that turns (seed, global trajectory index) into u0 and p. The
oracle (tests) and the GPU path both receive the arrays produced here; the
product also ships an on-device re-implementation of the same recipe
(``ens_generate_inputs``), which tests check bit-for-bit against this module.

Generator: SplitMix64 (Steele, Lea, Flood 2014) on a counter
    h = mix64(seed + (8·gidx + j + 1)·0x9E3779B97F4A7C15)   (mod 2^64)
    U = ((h >> 12) + 0.5)·2^-52                              (exact, in (0,1))
Recipes (all arithmetic in fp64, no contraction, then one cast to T):
    random10  : p_j = p̄_j · (1.0 + 0.1·(2U_j − 1))   "random p around p̄" (configs C1, C3, C5)
    rho_sweep : p = (10, 21·(g+1)/N_total, 8/3)        Lorenz ρ sweep over (0, 21]
    const     : p = p̄ broadcast                        SDE ensembles share p
u0 is the model's fixed ū0 for every trajectory.
Layout: SoA, u0[n][N], p[m][N] (trajectory fastest), the paper's U and P
matrices.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)

# p̄ and ū0 per model (P:634-642 Lorenz — BASELINE configs use ρ=28; P:668-679
# Robertson; P:684-688 GBM; DESIGN R9 stochastic Lorenz noise scale s=0.1).
MODELS = {
    "lorenz":         dict(pbar=(10.0, 28.0, 8.0 / 3.0), u0=(1.0, 0.0, 0.0)),
    "robertson":      dict(pbar=(0.04, 3e7, 1e4), u0=(1.0, 0.0, 0.0)),
    "lorenz_sde_add": dict(pbar=(10.0, 28.0, 8.0 / 3.0, 0.1), u0=(1.0, 0.0, 0.0)),
    "lorenz_sde_mul": dict(pbar=(10.0, 28.0, 8.0 / 3.0, 0.1), u0=(1.0, 0.0, 0.0)),
    "gbm":            dict(pbar=(1.5, 0.01), u0=(0.1, 0.1, 0.1)),
    "expdecay":       dict(pbar=(1.0,), u0=(1.0,)),
    "harmonic":       dict(pbar=(1.0,), u0=(1.0, 0.0)),
    # σ-factor CRN: p = (S, D, τ, ν0, n, η); Table 5 ranges; u0 = ν0
    "crn":            dict(pbar=(1.0, 1.0, 1.0, 0.1, 3.0, 0.05), u0=(0.1, 0.1, 0.1, 0.1),
                           lo=(0.1, 0.1, 0.1, 0.01, 2.0, 0.001), hi=(100.0, 100.0, 100.0, 0.2, 4.0, 0.1)),
}
RECIPES = {"random10": 0, "rho_sweep": 1, "const": 2, "grid": 3}
# stiff test suite, constants and initial states as printed
# bouncing ball: p = (g, e), dropped from rest at x = 50 (DESIGN R18)
MODELS["ball"] = dict(pbar=(9.8, 0.85), u0=(50.0, 0.0))
MODELS["orego"] = dict(pbar=(77.27, 8.375e-6, 0.161), u0=(1.0, 2.0, 3.0))
MODELS["hires"] = dict(pbar=(1.71, 0.43, 8.32, 0.0007, 8.75, 10.03, 0.035, 1.12, 1.745, 280.0, 0.69, 1.81),
                       u0=(1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0057))
MODELS["pollu"] = dict(pbar=(0.35, 26.6, 12300.0, 0.00086, 0.00082, 15000.0, 0.00013, 24000.0, 16500.0, 9000.0,
                             0.022, 12000.0, 1.88, 16300.0, 4.8e6, 0.00035, 0.0175, 1.0e8, 4.44e11, 1240.0, 2.1,
                             5.78, 0.0474, 1780.0, 3.12),
                       u0=(0.0, 0.2, 0.0, 0.04, 0.0, 0.0, 0.1, 0.3, 0.017, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0,
                           0.007, 0.0, 0.0, 0.0))


def grid_levels(n_total: int, m: int = 6) -> int:
    """Smallest L >= 2 with L^m >= n_total (levels per parameter of the grid recipe)."""
    L = 2
    while L**m < n_total:
        L += 1
    return L


NP_DTYPE = {"f32": np.float32, "f64": np.float64}


def mix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def uniform(seed: int, gidx: np.ndarray, j: int) -> np.ndarray:
    """U ∈ (0,1) for parameter slot j of trajectories gidx (fp64, exact)."""
    g = np.asarray(gidx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = g * np.uint64(8) + np.uint64(j + 1)
        h = mix64(np.uint64(seed) + ctr * GOLDEN)
    return ((h >> np.uint64(12)).astype(np.float64) + 0.5) * 2.0**-52


def global_indices(N: int, index_offset: int = 0, chunk_len: int = 0, chunk_stride: int = 0) -> np.ndarray:
    """Global index of local trajectory i (contiguous, or block-cyclic when chunk_len > 0)."""
    i = np.arange(N, dtype=np.int64)
    if chunk_len > 0:
        return index_offset + (i // chunk_len) * chunk_stride + i % chunk_len
    return index_offset + i


def make_inputs(model: str, recipe: str, N: int, *, seed: int = 0, dtype: str = "f64", index_offset: int = 0,
                N_total: int | None = None, chunk_len: int = 0, chunk_stride: int = 0):
    """Returns (u0 [n][N], p [m][N] or [m] for 'const') as numpy arrays in T."""
    spec = MODELS[model]
    pbar = np.array(spec["pbar"], dtype=np.float64)
    n, m = len(spec["u0"]), len(pbar)
    T = NP_DTYPE[dtype]
    u0 = np.empty((n, N), dtype=T)
    for c in range(n):
        u0[c, :] = T(spec["u0"][c])
    if recipe == "const":
        return u0, pbar.astype(T)
    g = global_indices(N, index_offset, chunk_len, chunk_stride)
    p = np.empty((m, N), dtype=np.float64)
    if recipe == "random10":
        for j in range(m):
            U = uniform(seed, g, j)
            p[j] = pbar[j] * (1.0 + 0.1 * (2.0 * U - 1.0))
    elif recipe == "grid":
        # Cartesian product of uniformly spaced levels ("each of the parameters is uniformly
        # sampled and the set of the Cartesian products … is simulated"); parameter 0 varies fastest
        if model != "crn":
            raise ValueError("grid is the CRN recipe")
        L = grid_levels(N if N_total is None else N_total, m)
        lo, hi = spec["lo"], spec["hi"]
        r = g.astype(np.int64).copy()
        for j in range(m):
            d = r % L
            r //= L
            p[j] = (hi[j] - lo[j]) * (d.astype(np.float64) / float(L - 1)) + lo[j]
        for c in range(n):
            u0[c, :] = p[3].astype(T)                      # u0 = ν0
    elif recipe == "rho_sweep":
        if model != "lorenz":
            raise ValueError("rho_sweep is a Lorenz recipe")
        Nt = float(N if N_total is None else N_total)
        p[0] = 10.0
        p[1] = (21.0 * (g + 1).astype(np.float64)) / Nt
        p[2] = 8.0 / 3.0
    else:
        raise ValueError(recipe)
    return u0, p.astype(T)
