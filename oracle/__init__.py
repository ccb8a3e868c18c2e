"""CPU oracle for the ensemble ODE/SDE solver — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded reference written from arXiv 2304.06835 (see the
header of oracle.cpp for citations and pins). Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` legs may import this package.
The product package ``paper_2304_06835_b200`` never imports it.

This module is ctypes marshalling only: every arithmetic step lives in
oracle.cpp.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "oracle.cpp"
_LIB = _HERE / "liboracle.so"

MODELS = {"lorenz": 0, "robertson": 1, "lorenz_sde_add": 2, "lorenz_sde_mul": 3, "gbm": 4,
          "expdecay": 5, "harmonic": 6, "crn": 7, "orego": 8, "hires": 9, "pollu": 10,
          "ball": 11}
ALGS = {"tsit5": 0, "rosenbrock23": 1, "em": 2, "siea": 3, "rodas4": 4, "vern7": 5, "rodas5": 6, "vern9": 7,
         "rodas5p": 8}
DTYPES = {"f32": 0, "f64": 1}
NP_DTYPE = {"f32": np.float32, "f64": np.float64}

CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> Path:
    """Compile liboracle.so (plain g++, no contraction, no fast-math)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["g++", *CXXFLAGS, "-o", str(tmp), str(_SRC)])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        vp, i32, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.orc_model_dims.argtypes = [i32, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.orc_rhs.argtypes = [i32, i32, vp, vp, dbl, vp]
        L.orc_jac.argtypes = [i32, i32, vp, vp, dbl, vp]
        L.orc_diffusion.argtypes = [i32, i32, vp, vp, dbl, vp]
        L.orc_tsit5_tableau.argtypes = [vp, vp, vp, vp]
        L.orc_ros23_consts.argtypes = [vp, vp]
        L.orc_rodas4_tableau.argtypes = [vp, vp, vp, vp]
        L.orc_vern7_tableau.argtypes = [vp, vp, vp, vp]
        L.orc_rodas5_tableau.argtypes = [vp, vp, vp]
        L.orc_rodas5p_tableau.argtypes = [vp, vp, vp]
        L.orc_vern9_tableau.argtypes = [vp, vp, vp, vp]
        L.orc_controller.argtypes = [i32, vp]
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_pi.argtypes = [i32, i32, dbl, dbl, ctypes.POINTER(dbl)]
        L.orc_pi.restype = dbl
        L.orc_log2.argtypes = [i32, dbl]
        L.orc_log2.restype = dbl
        L.orc_exp2.argtypes = [i32, dbl]
        L.orc_exp2.restype = dbl
        L.orc_sincospi.argtypes = [i32, dbl, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
        L.orc_error_q2.argtypes = [i32, vp, vp, vp, dbl, dbl]
        L.orc_error_q2.restype = dbl
        L.orc_uniforms.argtypes = [i32, vp, vp]
        L.orc_normals.argtypes = [i32, u64, u64, i64, i64, i32, vp]
        L.orc_fixed_grid.argtypes = [dbl, dbl, dbl, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
        L.orc_lu_solve.argtypes = [i32, i32, vp, vp, vp]
        L.orc_set_plain.argtypes = [i32]
        L.orc_set_plain.restype = i32
        L.orc_ros23_step.argtypes = [i32, vp, dbl, dbl, vp, vp, vp]
        L.orc_solve.argtypes = [i32, i32, i32, i64, vp, vp, i32, vp, dbl, dbl, dbl, i32, dbl, dbl, i64, u64,
                                vp, i32, vp, vp, vp, vp]
        L.orc_stats.argtypes = [i32, i64, i32, i32, vp, vp, vp, vp, ctypes.POINTER(i64)]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def model_dims(model: str):
    n, m, nw = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    if lib().orc_model_dims(MODELS[model], ctypes.byref(n), ctypes.byref(m), ctypes.byref(nw)):
        raise ValueError(model)
    return n.value, m.value, nw.value


def rhs(model: str, u, p, t=0.0, dtype="f64"):
    dt = NP_DTYPE[dtype]
    u = np.ascontiguousarray(u, dt); p = np.ascontiguousarray(p, dt)
    f = np.zeros_like(u)
    lib().orc_rhs(MODELS[model], DTYPES[dtype], _p(u), _p(p), t, _p(f))
    return f


def jac(model: str, u, p, t=0.0, dtype="f64"):
    dt = NP_DTYPE[dtype]
    u = np.ascontiguousarray(u, dt); p = np.ascontiguousarray(p, dt)
    J = np.zeros((u.size, u.size), dt)
    lib().orc_jac(MODELS[model], DTYPES[dtype], _p(u), _p(p), t, _p(J))
    return J


def diffusion(model: str, u, p, t=0.0, dtype="f64"):
    dt = NP_DTYPE[dtype]
    u = np.ascontiguousarray(u, dt); p = np.ascontiguousarray(p, dt)
    b = np.zeros_like(u)
    lib().orc_diffusion(MODELS[model], DTYPES[dtype], _p(u), _p(p), t, _p(b))
    return b


def tsit5_tableau():
    c = np.zeros(7); A = np.zeros((7, 7)); bt = np.zeros(7); r = np.zeros((7, 4))
    lib().orc_tsit5_tableau(_p(c), _p(A), _p(bt), _p(r))
    return c, A, bt, r


def ros23_consts():
    d = np.zeros(1); e = np.zeros(1)
    lib().orc_ros23_consts(_p(d), _p(e))
    return float(d[0]), float(e[0])


def rodas4_tableau():
    """(gamma, A[6,6], C[6,6], D[2,5]) of the Rodas4 W-form (DESIGN R20)."""
    g = np.zeros(1); A = np.zeros((6, 6)); C = np.zeros((6, 6)); D = np.zeros((2, 5))
    lib().orc_rodas4_tableau(_p(g), _p(A), _p(C), _p(D))
    return float(g[0]), A, C, D


def vern7_tableau():
    """(c[10], A[10,10], b[10], btilde[10]) of Vern7 (DESIGN R21)."""
    c = np.zeros(10); A = np.zeros((10, 10)); b = np.zeros(10); bt = np.zeros(10)
    lib().orc_vern7_tableau(_p(c), _p(A), _p(b), _p(bt))
    return c, A, b, bt


def vern9_tableau():
    """(c[16], A[16,16], b[16], btilde[16]) of Vern9 (DESIGN R21)."""
    c = np.zeros(16); A = np.zeros((16, 16)); b = np.zeros(16); bt = np.zeros(16)
    lib().orc_vern9_tableau(_p(c), _p(A), _p(b), _p(bt))
    return c, A, b, bt


def rodas5_tableau():
    """(gamma, A[8,8], C[8,8]) of Rodas5 in W-form (DESIGN R22)."""
    g = np.zeros(1); A = np.zeros((8, 8)); C = np.zeros((8, 8))
    lib().orc_rodas5_tableau(_p(g), _p(A), _p(C))
    return float(g[0]), A, C


def rodas5p_tableau():
    """(gamma, A[8,8], C[8,8]) of Rodas5P in W-form (DESIGN R23)."""
    g = np.zeros(1); A = np.zeros((8, 8)); C = np.zeros((8, 8))
    lib().orc_rodas5p_tableau(_p(g), _p(A), _p(C))
    return float(g[0]), A, C


def controller(alg: str):
    out = np.zeros(6)
    lib().orc_controller(ALGS[alg], _p(out))
    return dict(zip(["beta1", "beta2", "eta", "qmin_inv", "qmax_inv", "qold_floor"], out.tolist()))


def pi_step(alg: str, accept: bool, h: float, q2: float, lq_old: float):
    """PI controller (fp64, exponent domain, DESIGN R2): returns (h_new, log2 q_old after the step)."""
    lo = ctypes.c_double(lq_old)
    hn = lib().orc_pi(ALGS[alg], int(accept), h, q2, ctypes.byref(lo))
    return hn, lo.value


def log2_spec(x: float, dtype="f64") -> float:
    return lib().orc_log2(DTYPES[dtype], float(x))


def exp2_spec(z: float, dtype="f64") -> float:
    return lib().orc_exp2(DTYPES[dtype], float(z))


def sincospi_spec(t: float, dtype="f64"):
    """(sin πt, cos πt) by the Box–Muller polynomial (DESIGN R8)."""
    s, c = ctypes.c_double(), ctypes.c_double()
    lib().orc_sincospi(DTYPES[dtype], float(t), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def error_q2(E, u, unew, abstol, reltol):
    """Squared error proportion q² (Eq. q, RMS reading)."""
    E = np.ascontiguousarray(E, np.float64); u = np.ascontiguousarray(u, np.float64)
    un = np.ascontiguousarray(unew, np.float64)
    return lib().orc_error_q2(E.size, _p(E), _p(u), _p(un), abstol, reltol)


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32); k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def uniforms(words, dtype="f32"):
    w = np.ascontiguousarray(words, np.uint32)
    out = np.zeros(4 if dtype == "f32" else 2, NP_DTYPE[dtype])
    lib().orc_uniforms(DTYPES[dtype], _p(w), _p(out))
    return out


def normals(seed: int, gidx: int, step0: int, count: int, dtype="f64", nw: int = 3):
    out = np.zeros((count, nw), NP_DTYPE[dtype])
    lib().orc_normals(DTYPES[dtype], seed, gidx, step0, count, nw, _p(out))
    return out


def set_plain(on: bool) -> bool:
    """Test-only: evaluate the PI controller literally with libm pow and
    Box–Muller with libm log/sin/cos (True), or in the canonical forms of
    DESIGN R2 / R8 that the kernels follow (False, the default). Returns the
    previous mode."""
    return bool(lib().orc_set_plain(int(bool(on))))


class plain_mode:
    """Context manager: ``with oracle.plain_mode(): ...`` runs the oracle in plain mode."""

    def __enter__(self):
        self._prev = set_plain(True)
        return self

    def __exit__(self, *exc):
        set_plain(self._prev)
        return False


def ros23_step(model: str, u, p, t: float, h: float):
    """One fp64 Rosenbrock23 step from u (F0 = f(u)): (u_new, E), or None if W is singular."""
    u = np.ascontiguousarray(u, np.float64); p = np.ascontiguousarray(p, np.float64)
    un = np.zeros_like(u); E = np.zeros_like(u)
    if lib().orc_ros23_step(MODELS[model], _p(p), float(t), float(h), _p(u), _p(un), _p(E)):
        return None
    return un, E


def fixed_grid(t0, tf, dt):
    ns, hl = ctypes.c_int64(), ctypes.c_double()
    lib().orc_fixed_grid(t0, tf, dt, ctypes.byref(ns), ctypes.byref(hl))
    return ns.value, hl.value


def lu_solve(A, b, dtype="f64"):
    dt = NP_DTYPE[dtype]
    A = np.ascontiguousarray(A, dt); b = np.ascontiguousarray(b, dt)
    x = np.zeros_like(b)
    if lib().orc_lu_solve(DTYPES[dtype], b.size, _p(A), _p(b), _p(x)):
        return None
    return x


def solve(model: str, alg: str, u0, p, tspan, dt, *, dtype="f64", adaptive=False, abstol=1e-6, reltol=1e-3,
          max_steps=0, seed=0, saveat=None, p_broadcast=False, gidx=None):
    """Solve an ensemble trajectory by trajectory. u0: [n][N], p: [m][N] (or [m] if
    p_broadcast). Returns (u_out [max(k,1)][n][N], retcode, n_accept, n_reject)."""
    npd = NP_DTYPE[dtype]
    u0 = np.ascontiguousarray(u0, npd)
    p = np.ascontiguousarray(p, npd)
    n, N = u0.shape
    sa = None if saveat is None else np.ascontiguousarray(saveat, np.float64)
    k = 0 if sa is None else sa.size
    out = np.empty((max(k, 1), n, N), npd)
    rc = np.empty(N, np.int32); na = np.empty(N, np.int32); nr = np.empty(N, np.int32)
    g = None if gidx is None else np.ascontiguousarray(gidx, np.uint64)
    err = lib().orc_solve(MODELS[model], ALGS[alg], DTYPES[dtype], N, _p(u0), _p(p), int(p_broadcast), _p(g),
                          float(tspan[0]), float(tspan[1]), float(dt), int(adaptive), float(abstol),
                          float(reltol), int(max_steps), int(seed), _p(sa), k, _p(out), _p(rc), _p(na), _p(nr))
    if err:
        raise RuntimeError(f"orc_solve failed ({err})")
    return out, rc, na, nr


def stats(x, mask=None):
    """Two-pass long-double mean/unbiased variance over axis -1 of x [k][n][N]."""
    x = np.ascontiguousarray(x)
    dtype = "f32" if x.dtype == np.float32 else "f64"
    k, n, N = x.shape
    mean = np.zeros((k, n)); var = np.zeros((k, n))
    m = None if mask is None else np.ascontiguousarray(mask, np.int32)
    cnt = ctypes.c_int64()
    lib().orc_stats(DTYPES[dtype], N, k, n, _p(x), _p(m), _p(mean), _p(var), ctypes.byref(cnt))
    return mean, var, cnt.value
