"""B200-native ensemble ODE/SDE solver (arXiv 2304.06835's EnsembleGPUKernel hot path).

Thin Python binding over the C ABI in include/ens.h (libens.so, sm_100a):
argument marshalling only — every step of the solve runs in the CUDA kernels.
PyTorch supplies device memory and streams. There is no CPU fallback: if the
extension is missing this module raises instead of computing anything.

Layout: SoA, trajectory fastest — u0 is [n, N], p is [m, N] (or [m] when
broadcast), saved states are [k, n, N] (the paper's U / P matrices).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import torch

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "libens.so"

MODELS = {"lorenz": 0, "robertson": 1, "lorenz_sde_add": 2, "lorenz_sde_mul": 3, "gbm": 4, "expdecay": 5,
          "harmonic": 6, "crn": 7, "orego": 8, "hires": 9, "pollu": 10, "ball": 11}
ALGS = {"tsit5": 0, "rosenbrock23": 1, "em": 2, "siea": 3, "rodas4": 4, "vern7": 5, "rodas5": 6, "vern9": 7,
         "rodas5p": 8}
DTYPES = {torch.float32: 0, torch.float64: 1}
RECIPES = {"random10": 0, "rho_sweep": 1, "const": 2, "grid": 3}
RETCODES = {0: "Success", 1: "MaxIters", 2: "DtLessThanMin", 3: "Diverged", 4: "Singular"}


class EnsError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {status_string(status)} (status {status})")
        self.status = status


class _Options(ctypes.Structure):
    _fields_ = [("adaptive", ctypes.c_int32), ("abstol", ctypes.c_double), ("reltol", ctypes.c_double),
                ("max_steps", ctypes.c_int64), ("seed", ctypes.c_uint64), ("saveat", ctypes.c_void_p),
                ("n_saveat", ctypes.c_int32), ("p_broadcast", ctypes.c_int32), ("want_stats", ctypes.c_int32),
                ("refill", ctypes.c_int32), ("index_offset", ctypes.c_int64), ("chunk_len", ctypes.c_int64),
                ("chunk_stride", ctypes.c_int64), ("out_ld", ctypes.c_int64), ("bulk_saves", ctypes.c_int32)]


class _Output(ctypes.Structure):
    _fields_ = [("u_out", ctypes.c_void_p), ("retcode", ctypes.c_void_p), ("n_accept", ctypes.c_void_p),
                ("n_reject", ctypes.c_void_p), ("stats", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t)]


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libens.so (built by __graft_entry__.build() / _build.py). Raises if absent."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"{_LIB_PATH} is missing: build it with `python -m paper_2304_06835_b200._build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(str(_LIB_PATH))
        vp, i32, i64, u64, dbl, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_double, ctypes.c_size_t)
        L.ens_model_dims.argtypes = [i32, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.ens_model_dims.restype = i32
        L.ens_workspace_bytes.argtypes = [i32, i32, i32, i64, ctypes.POINTER(_Options)]
        L.ens_workspace_bytes.restype = sz
        L.ensemble_solve.argtypes = [i32, i32, i32, i64, vp, vp, dbl, dbl, dbl, ctypes.POINTER(_Options),
                                     ctypes.POINTER(_Output), vp]
        L.ensemble_solve.restype = i32
        L.ensemble_solve_host.argtypes = [i32, i32, i32, i64, vp, vp, dbl, dbl, dbl, ctypes.POINTER(_Options),
                                          vp, vp, vp, vp, vp, vp, vp, sz, i32, vp]
        L.ensemble_solve_host.restype = i32
        L.ens_generate_inputs.argtypes = [i32, i32, i32, u64, i64, i64, ctypes.POINTER(_Options), vp, vp, vp]
        L.ens_generate_inputs.restype = i32
        L.ens_ensemble_stats.argtypes = [i32, vp, i64, i64, i32, vp, vp, sz, vp]
        L.ens_ensemble_stats.restype = i32
        L.ens_stats_workspace_bytes.argtypes = [i64, i32]
        L.ens_stats_workspace_bytes.restype = sz
        L.ens_stats_finalize.argtypes = [vp, i32, i32, vp, vp, vp]
        L.ens_stats_finalize.restype = i32
        L.ens_stats_merge.argtypes = [vp, i32, i32, i32, vp, vp]
        L.ens_stats_merge.restype = i32
        L.ens_sde_noise.argtypes = [i32, u64, i64, i64, i64, i32, ctypes.POINTER(_Options), vp, vp, vp]
        L.ens_sde_noise.restype = i32
        L.ens_philox4x32_10.argtypes = [vp, vp, vp, i64, vp]
        L.ens_philox4x32_10.restype = i32
        L.ens_check_fast_paths.argtypes = [vp, vp]
        L.ens_check_fast_paths.restype = i32
        L.ens_status_string.argtypes = [i32]
        L.ens_status_string.restype = ctypes.c_char_p
        L.ens_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


EXPORTS = ["ens_model_dims", "ens_workspace_bytes", "ensemble_solve", "ensemble_solve_host", "ens_generate_inputs",
           "ens_ensemble_stats", "ens_stats_workspace_bytes", "ens_stats_finalize", "ens_stats_merge", "ens_sde_noise", "ens_philox4x32_10", "ens_check_fast_paths",
           "ens_status_string", "ens_version"]


def status_string(status: int) -> str:
    return lib().ens_status_string(status).decode()


def model_dims(model: str):
    n, m, nw = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    st = lib().ens_model_dims(MODELS[model], ctypes.byref(n), ctypes.byref(m), ctypes.byref(nw))
    if st:
        raise EnsError(st, "ens_model_dims")
    return n.value, m.value, nw.value


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream) -> Optional[int]:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _options(adaptive, abstol, reltol, max_steps, seed, saveat_buf, p_broadcast, stats, refill, index_offset,
             chunk_len, chunk_stride) -> _Options:
    o = _Options()
    o.adaptive = int(adaptive)
    o.abstol = float(abstol); o.reltol = float(reltol)
    o.max_steps = int(max_steps); o.seed = int(seed)
    if saveat_buf is not None:
        o.saveat = saveat_buf.ctypes.data
        o.n_saveat = len(saveat_buf)
    o.p_broadcast = int(p_broadcast); o.want_stats = int(stats); o.refill = int(refill)
    o.index_offset = int(index_offset); o.chunk_len = int(chunk_len); o.chunk_stride = int(chunk_stride)
    return o


@dataclass
class Solution:
    u: Optional[torch.Tensor]          # [k, n, N] (k = len(saveat)) or [n, N]
    retcode: torch.Tensor              # [N] int32
    n_accept: torch.Tensor             # [N] int32
    n_reject: torch.Tensor             # [N] int32
    stats: Optional[torch.Tensor]      # [max(k,1), n, 3] fp64 (count, mean, M2)

    def mean_var(self):
        """(mean, unbiased variance) from the fused statistics, on device (ens_stats_finalize)."""
        return stats_finalize(self.stats)


class Workspace:
    """Reusable device workspace (caller-owned scratch for ensemble_solve)."""

    def __init__(self, nbytes: int, device):
        self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)

    def ensure(self, nbytes: int):
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=self.buf.device)
        return self.buf


def solve(model: str, alg: str, u0: torch.Tensor, p: torch.Tensor, tspan: Sequence[float], dt: float, *,
          adaptive: bool = False, abstol: float = 1e-6, reltol: float = 1e-3, saveat: Optional[Sequence[float]] = None,
          max_steps: int = 0, seed: int = 0, stats: bool = False, refill: bool = False, index_offset: int = 0,
          chunk_len: int = 0, chunk_stride: int = 0, store_states: bool = True, workspace: Optional[Workspace] = None,
          out: Optional[Solution] = None, stream=None, bulk_saves: bool = False) -> Solution:
    """ensemble_solve on device tensors. u0 [n, N], p [m, N] (or [m]: broadcast), same float dtype."""
    import numpy as np
    if not u0.is_cuda or not p.is_cuda:
        raise ValueError("u0 and p must be CUDA tensors (no CPU path)")
    if u0.dtype != p.dtype or u0.dtype not in DTYPES:
        raise ValueError("u0 and p must share dtype float32 or float64")
    u0 = u0.contiguous(); p = p.contiguous()
    n, N = u0.shape
    nm, m, nw = model_dims(model)
    if n != nm:
        raise ValueError(f"{model}: u0 must be [{nm}, N]")
    p_broadcast = p.dim() == 1
    sa = None if saveat is None else np.ascontiguousarray(np.asarray(saveat, dtype=np.float64))
    k = 0 if sa is None else sa.size
    opt = _options(adaptive, abstol, reltol, max_steps, seed, sa, p_broadcast, stats, refill, index_offset,
                   chunk_len, chunk_stride)
    opt.bulk_saves = int(bool(bulk_saves))
    dev = u0.device
    if out is None:
        shape = (k, n, N) if k else (n, N)
        u_out = torch.empty(shape, dtype=u0.dtype, device=dev) if (store_states or alg not in ("em", "siea")) else None
        out = Solution(u=u_out, retcode=torch.empty(N, dtype=torch.int32, device=dev),
                       n_accept=torch.empty(N, dtype=torch.int32, device=dev),
                       n_reject=torch.empty(N, dtype=torch.int32, device=dev),
                       stats=torch.empty((max(k, 1), n, 3), dtype=torch.float64, device=dev) if stats else None)
    if out.u is not None:
        # u_out may be a column slice of a larger [k][n][L] / [n][L] array (e.g. a peer GPU's gather
        # buffer): rows of L elements, trajectory-contiguous
        u = out.u
        if u.dtype != u0.dtype or u.shape[-1] != N or u.stride(-1) != 1:
            raise ValueError("out.u must have the input dtype, N trajectories in its last dimension, stride 1")
        ld_rows = u.stride(-2)
        if u.dim() == 3 and u.stride(0) != u.shape[1] * ld_rows:
            raise ValueError("out.u: save points must be stacked with the row stride")
        opt.out_ld = 0 if ld_rows == N else int(ld_rows)
    L = lib()
    wsb = L.ens_workspace_bytes(MODELS[model], ALGS[alg], DTYPES[u0.dtype], N, ctypes.byref(opt))
    if workspace is None:
        workspace = Workspace(wsb, dev)
    ws = workspace.ensure(wsb)
    o = _Output(u_out=_ptr(out.u), retcode=_ptr(out.retcode), n_accept=_ptr(out.n_accept),
                n_reject=_ptr(out.n_reject), stats=_ptr(out.stats), workspace=_ptr(ws), workspace_bytes=ws.numel())
    with torch.cuda.device(dev):
        st = L.ensemble_solve(MODELS[model], ALGS[alg], DTYPES[u0.dtype], N, _ptr(u0), _ptr(p), float(tspan[0]),
                              float(tspan[1]), float(dt), ctypes.byref(opt), ctypes.byref(o), _stream_ptr(stream))
    if st:
        raise EnsError(st, "ensemble_solve")
    if stream is not None and stream != torch.cuda.current_stream(dev):
        # the kernel runs on `stream`: keep the caching allocator from handing this call's
        # temporaries (workspace, contiguous copies of u0 / p, outputs) to other work on the
        # current stream before the kernel is done with them
        for t in (u0, p, ws, out.u, out.retcode, out.n_accept, out.n_reject, out.stats):
            if t is not None and t.is_cuda and t.device == dev:
                t.record_stream(stream)
    return out


def solve_host(model: str, alg: str, u0_host: torch.Tensor, p_host: torch.Tensor, tspan, dt, *, device=None,
               adaptive=False, abstol=1e-6, reltol=1e-3, saveat=None, max_steps=0, refill=False, n_chunks=4,
               seed=0, index_offset=0, staging=None, u_out_host=None, retcode_host=None, stream=None):
    """ensemble_solve_host: host (pinned) inputs → chunked H2D / solve / D2H overlapped → host outputs."""
    import numpy as np
    dev = torch.device(device or "cuda")
    n, N = u0_host.shape
    p_broadcast = p_host.dim() == 1
    sa = None if saveat is None else np.ascontiguousarray(np.asarray(saveat, dtype=np.float64))
    k = 0 if sa is None else sa.size
    opt = _options(adaptive, abstol, reltol, max_steps, seed, sa, p_broadcast, False, refill, index_offset, 0, 0)
    L = lib()
    dt_ = u0_host.dtype
    wsb = L.ens_workspace_bytes(MODELS[model], ALGS[alg], DTYPES[dt_], N, ctypes.byref(opt))
    if staging is None:
        staging = dict(u0=torch.empty_like(u0_host, device=dev), p=torch.empty_like(p_host, device=dev),
                       u=torch.empty((max(k, 1), n, N), dtype=dt_, device=dev),
                       rc=torch.empty(N, dtype=torch.int32, device=dev),
                       ws=torch.empty(wsb, dtype=torch.uint8, device=dev))
    if u_out_host is None:
        u_out_host = torch.empty((max(k, 1), n, N), dtype=dt_, pin_memory=True)
    if retcode_host is None:
        retcode_host = torch.empty(N, dtype=torch.int32, pin_memory=True)
    with torch.cuda.device(dev):
        st = L.ensemble_solve_host(MODELS[model], ALGS[alg], DTYPES[dt_], N, _ptr(u0_host), _ptr(p_host),
                                   float(tspan[0]), float(tspan[1]), float(dt), ctypes.byref(opt), _ptr(staging["u0"]),
                                   _ptr(staging["p"]), _ptr(staging["u"]), _ptr(staging["rc"]), _ptr(u_out_host),
                                   _ptr(retcode_host), _ptr(staging["ws"]), staging["ws"].numel(), int(n_chunks),
                                   _stream_ptr(stream))
    if st:
        raise EnsError(st, "ensemble_solve_host")
    return (u_out_host if k else u_out_host[0]), retcode_host, staging


def generate_inputs(model: str, recipe: str, N: int, *, dtype=torch.float32, seed: int = 0, index_offset: int = 0,
                    N_total: int = 0, chunk_len: int = 0, chunk_stride: int = 0, device=None, stream=None):
    """ens_generate_inputs: on-device twin of synth/inputs.make_inputs (bit-identical)."""
    n, m, _ = model_dims(model)
    dev = torch.device(device or "cuda")
    u0 = torch.empty((n, N), dtype=dtype, device=dev)
    p = torch.empty((m,) if recipe == "const" else (m, N), dtype=dtype, device=dev)
    opt = _options(0, 0, 0, 0, 0, None, 0, 0, 0, index_offset, chunk_len, chunk_stride)
    with torch.cuda.device(dev):
        st = lib().ens_generate_inputs(MODELS[model], DTYPES[dtype], RECIPES[recipe], int(seed), int(N), int(N_total),
                                       ctypes.byref(opt), _ptr(u0), _ptr(p), _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_generate_inputs")
    return u0, p


def ensemble_stats(x: torch.Tensor, *, out: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                   stream=None, device=None) -> torch.Tensor:
    """ens_ensemble_stats: (count, mean, M2) over the last axis of x [..., N] (finite values only).
    Runs on `device`, else the device of `out`, else x's; x may live on a peer GPU (a PeerGather view),
    read over NVLink by the executing device."""
    N = x.shape[-1]
    rows = x.numel() // N
    # rows may sit `ld` apart (a slice of a wider array, e.g. a PeerGather view); anything else is densified
    ld = x.stride(-2) if x.dim() >= 2 else N
    uniform = x.stride(-1) == 1 and all(x.stride(d) == x.stride(d + 1) * x.shape[d + 1] for d in range(x.dim() - 2))
    if not uniform or ld < N:
        x = x.contiguous()
        ld = N
    dev = torch.device(device) if device is not None else (out.device if out is not None else x.device)
    if out is None:
        out = torch.empty((*x.shape[:-1], 3), dtype=torch.float64, device=dev)
    L = lib()
    wsb = L.ens_stats_workspace_bytes(N, rows)
    if workspace is None:
        workspace = Workspace(wsb, dev)
    ws = workspace.ensure(wsb)
    with torch.cuda.device(dev):
        st = L.ens_ensemble_stats(DTYPES[x.dtype], _ptr(x), N, int(ld), rows, _ptr(out), _ptr(ws), ws.numel(),
                                  _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_ensemble_stats")
    return out


def stats_finalize(stats: torch.Tensor, stream=None):
    k, n, _ = stats.shape
    mean = torch.empty((k, n), dtype=torch.float64, device=stats.device)
    var = torch.empty_like(mean)
    with torch.cuda.device(stats.device):
        st = lib().ens_stats_finalize(_ptr(stats), k, n, _ptr(mean), _ptr(var), _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_stats_finalize")
    return mean, var


def stats_merge(gathered: torch.Tensor, stream=None) -> torch.Tensor:
    """Fixed-rank-order Chan merge of [R, k, n, 3] per-rank statistics (device)."""
    R, k, n, _ = gathered.shape
    merged = torch.empty((k, n, 3), dtype=torch.float64, device=gathered.device)
    with torch.cuda.device(gathered.device):
        st = lib().ens_stats_merge(_ptr(gathered.contiguous()), R, k, n, _ptr(merged), _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_stats_merge")
    return merged


def sde_noise(N: int, nsteps: int, *, seed: int, dtype=torch.float32, step0: int = 0, index_offset: int = 0,
              chunk_len: int = 0, chunk_stride: int = 0, nw: int = 3, device=None, stream=None):
    """ens_sde_noise: (Philox words [ncalls, 4, N] uint32-as-int32 of the stream's calls
    c0 = nw·step0 // PER …, normals [nsteps, nw, N]); PER = 4 (fp32) or 2 (fp64)."""
    dev = torch.device(device or "cuda")
    per = 4 if dtype == torch.float32 else 2
    c0 = nw * step0 // per
    ncalls = -(-(nw * (step0 + nsteps)) // per) - c0
    words = torch.empty((ncalls, 4, N), dtype=torch.int32, device=dev)
    z = torch.empty((nsteps, nw, N), dtype=dtype, device=dev)
    opt = _options(0, 0, 0, 0, 0, None, 0, 0, 0, index_offset, chunk_len, chunk_stride)
    with torch.cuda.device(dev):
        st = lib().ens_sde_noise(DTYPES[dtype], int(seed), int(N), int(step0), int(nsteps), int(nw),
                                 ctypes.byref(opt), _ptr(words), _ptr(z), _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_sde_noise")
    return words, z


def check_fast_paths(device=None):
    """ens_check_fast_paths: (mismatches of the log2 quotient over fp32 m in [√½, √2),
    mismatches of the Box–Muller sqrt over fp32 x in [1e-7, 64)) against IEEE division / sqrt."""
    dev = torch.device(device or "cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        st = lib().ens_check_fast_paths(_ptr(cnt), None)
    if st:
        raise EnsError(st, "ens_check_fast_paths")
    return tuple(int(v) for v in cnt.tolist())


def philox4x32_10(ctr: torch.Tensor, key: torch.Tensor, stream=None) -> torch.Tensor:
    """ens_philox4x32_10 on device int32 tensors ctr [N,4], key [N,2] (bit patterns as uint32)."""
    out = torch.empty_like(ctr)
    with torch.cuda.device(ctr.device):
        st = lib().ens_philox4x32_10(_ptr(ctr.contiguous()), _ptr(key.contiguous()), _ptr(out), ctr.shape[0],
                                     _stream_ptr(stream))
    if st:
        raise EnsError(st, "ens_philox4x32_10")
    return out


def workspace_bytes(model: str, alg: str, dtype, N: int, *, n_saveat=0, stats=False, adaptive=False, refill=False):
    opt = _Options()
    opt.n_saveat = n_saveat; opt.want_stats = int(stats); opt.adaptive = int(adaptive); opt.refill = int(refill)
    return lib().ens_workspace_bytes(MODELS[model], ALGS[alg], DTYPES[dtype], int(N), ctypes.byref(opt))
