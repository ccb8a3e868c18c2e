// api.cu — C ABI of the ensemble solver (include/ens.h): argument validation,
// workspace layout, dispatch over the template instances <Model, T, alg,
// adaptive, saveat, scheduler>, launch configuration, host end-to-end pipeline.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/ens.h"
#include "common.cuh"
#include "em.cuh"
#include "inputs.cuh"
#include "launch.cuh"
#include "stats.cuh"

using namespace ens;

int ens::sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Occupancy-tuned block sizes (launch.cuh::occupancy_block), cached per (kernel, start size).
namespace {
std::mutex g_block_mu;
std::map<std::pair<const void*, int>, int> g_block_cache;
}  // namespace
int ens::cached_block(const void* kernel, int b0) {
  std::lock_guard<std::mutex> lk(g_block_mu);
  const auto it = g_block_cache.find({kernel, b0});
  return it == g_block_cache.end() ? 0 : it->second;
}
void ens::cache_block(const void* kernel, int b0, int b) {
  std::lock_guard<std::mutex> lk(g_block_mu);
  g_block_cache[{kernel, b0}] = b;
}

namespace {

constexpr int64_t kStatsChunk = 8192;

bool model_dims(int model, int* n, int* m, int* nw) {
  switch (model) {
    case ENS_LORENZ: case ENS_ROBERTSON: *n = 3; *m = 3; *nw = 0; return true;
    case ENS_LORENZ_SDE_ADD: case ENS_LORENZ_SDE_MUL: *n = 3; *m = 4; *nw = 3; return true;
    case ENS_GBM: *n = 3; *m = 2; *nw = 3; return true;
    case ENS_EXPDECAY: *n = 1; *m = 1; *nw = 0; return true;
    case ENS_HARMONIC: *n = 2; *m = 1; *nw = 0; return true;
    case ENS_CRN: *n = 4; *m = 6; *nw = 8; return true;
    case ENS_OREGO: *n = 3; *m = 3; *nw = 0; return true;
    case ENS_HIRES: *n = 8; *m = 12; *nw = 0; return true;
    case ENS_POLLU: *n = 20; *m = 25; *nw = 0; return true;
    case ENS_BALL: *n = 2; *m = 2; *nw = 0; return true;
  }
  return false;
}

inline bool is_sde_alg(int alg) { return alg == ENS_EM || alg == ENS_SIEA; }
// save points given as step-grid indices (DESIGN R11: EM / SIEA)
inline bool grid_saves(int alg, const ens_options*) { return is_sde_alg(alg); }
// fixed-step saves by save codes (fixed_save_codes): Tsit5 (interpolant) and the
// dense-output-by-substep methods Vern7 / Vern9 / Rodas5 / Rodas5P (DESIGN R24)
inline bool coded_saves(int alg, const ens_options* opt) {
  return !opt->adaptive && (alg == ENS_TSIT5 || alg == ENS_VERN7 || alg == ENS_VERN9 || alg == ENS_RODAS5 ||
                            alg == ENS_RODAS5P);
}
inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// DESIGN R3: fixed-step count and last step, in fp64.
void fixed_grid(double t0, double tf, double dt, int64_t* nsteps, double* h_last) {
  const double r = (tf - t0) / dt;
  const double rr = std::nearbyint(r);
  int64_t ns = (std::fabs(r - rr) <= 1e-9 * std::max(1.0, r)) ? (int64_t)rr : (int64_t)std::ceil(r);
  if (ns < 1) ns = 1;
  *nsteps = ns;
  *h_last = (tf - t0) - (double)(ns - 1) * dt;
}

struct Layout {
  size_t counter, tau, save_step, partial, partial2, total;
  int64_t nparts;
  int rows;
};

// Statistics computed inside the solve kernel from registers (no pass over the stored states).
bool fused_stats(int alg, const ens_options* opt) {
  return opt && opt->want_stats && alg == ENS_TSIT5 && !opt->adaptive && opt->n_saveat == 0;
}

Layout layout(int n, int alg, int dtype, int64_t N, const ens_options* opt) {
  Layout L{};
  const int k = opt ? std::max(0, opt->n_saveat) : 0;
  const size_t tsz = dtype == ENS_F32 ? 4 : 8;
  L.counter = 0;
  L.tau = 256;
  L.save_step = L.tau + align256(std::max(1, k) * tsz);
  L.partial = L.save_step + align256(std::max(1, k) * 8);
  L.rows = std::max(1, k) * n;
  const bool stats = opt && opt->want_stats;
  L.nparts = 0;
  // EM: one partial per solver block; sized for the smallest block (32) so the layout is device independent
  // fixed-step Tsit5 without saves: one partial per warp, fused into the solve (tsit5_fixed_kernel STATS)
  if (stats) L.nparts = (is_sde_alg(alg) || fused_stats(alg, opt)) ? cdiv(N, 32) : cdiv(N, kStatsChunk);
  L.partial2 = L.partial + align256((size_t)L.rows * (size_t)L.nparts * 3 * 8);
  // first-stage merge outputs (stats_fold_kernel) when there are many partials
  L.total = L.partial2 + align256((size_t)L.rows * (size_t)cdiv(L.nparts, 256 * kFold) * 3 * 8) + 256;
  return L;
}

// ---------------------------------------------------------------- dispatch --
// Kernel instances live in one translation unit per algorithm (launch.cuh).
template <class T>
ens_status dispatch(int model, int alg, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  switch (alg) {
    case ENS_TSIT5: return launch_tsit5<T>(model, a, opt, s);
    case ENS_ROSENBROCK23: return launch_ros23<T>(model, a, opt, s);
    case ENS_RODAS4: return launch_rodas4<T>(model, a, opt, s);
    case ENS_VERN7: return launch_vern7<T>(model, a, opt, s);
    case ENS_RODAS5: return launch_rodas5<T>(model, a, opt, s);
    case ENS_VERN9: return launch_vern9<T>(model, a, opt, s);
    case ENS_RODAS5P: return launch_rodas5p<T>(model, a, opt, s);
    case ENS_EM: case ENS_SIEA: return launch_sde<T>(model, alg, a, opt, s);
  }
  return ENS_E_INVALID_ARG;
}

// Validation shared by ensemble_solve and ensemble_solve_host.
ens_status validate(int model, int alg, int dtype, int64_t N, double t0, double tf, double dt,
                    const ens_options* opt, int* n_out) {
  int n, m, nw;
  if (!opt || N < 1 || !model_dims(model, &n, &m, &nw)) return ENS_E_INVALID_ARG;
  if (alg < ENS_TSIT5 || alg > ENS_RODAS5P || (dtype != ENS_F32 && dtype != ENS_F64)) return ENS_E_INVALID_ARG;
  if (opt->n_saveat < 0 || (opt->n_saveat > 0 && !opt->saveat)) return ENS_E_INVALID_ARG;
  if (opt->chunk_len < 0 || opt->index_offset < 0) return ENS_E_INVALID_ARG;
  if (opt->out_ld != 0 && opt->out_ld < N) return ENS_E_INVALID_ARG;
  const bool sde = nw > 0;
  if (sde != is_sde_alg(alg)) return ENS_E_ALG_MISMATCH;
  // events (DESIGN R18) are located on the adaptive Tsit5 interpolant only
  if (model == ENS_BALL && (alg != ENS_TSIT5 || !opt->adaptive)) return ENS_E_UNSUPPORTED;
  if (dtype == ENS_F32 && model == ENS_POLLU) return ENS_E_UNSUPPORTED;   // n = 20: fp64 stiff solvers only
  // explicit solvers keep all stages in registers; they are instantiated for n <= 8
  if (n > 8 && (alg == ENS_TSIT5 || alg == ENS_VERN7 || alg == ENS_VERN9)) return ENS_E_UNSUPPORTED;
  if (is_sde_alg(alg) && opt->adaptive) return ENS_E_ADAPTIVE_UNSUPPORTED;
  if (!std::isfinite(t0) || !std::isfinite(tf) || !std::isfinite(dt) || !(t0 < tf) || !(dt > 0))
    return ENS_E_BAD_TSPAN;
  if (opt->adaptive) {
    if (!std::isfinite(opt->abstol) || !std::isfinite(opt->reltol) || !(opt->abstol > 0) || !(opt->reltol >= 0))
      return ENS_E_BAD_TOLERANCE;
  }
  const int k = opt->n_saveat;
  for (int j = 0; j < k; ++j) {
    const double tj = opt->saveat[j];
    if (!std::isfinite(tj) || tj < t0 || tj > tf) return ENS_E_BAD_SAVEAT;
    if (j > 0 && !(tj > opt->saveat[j - 1])) return ENS_E_BAD_SAVEAT;
    if (j > 0) {   // strictly increasing also after the cast to T
      if (dtype == ENS_F32 && !((float)tj > (float)opt->saveat[j - 1])) return ENS_E_BAD_SAVEAT;
    }
  }
  *n_out = n;
  return ENS_OK;
}

// EM save points as grid indices (DESIGN R11): τ must be t0 + s·dt (s < nsteps) or tf.
bool em_save_steps(double t0, double tf, double dt, const double* sa, int k, std::vector<int64_t>& out) {
  int64_t nsteps; double hl;
  fixed_grid(t0, tf, dt, &nsteps, &hl);
  out.resize(k);
  for (int j = 0; j < k; ++j) {
    int64_t s;
    if (sa[j] == tf) s = nsteps;
    else {
      s = (int64_t)std::nearbyint((sa[j] - t0) / dt);
      if (s < 0 || s >= nsteps) return false;
      if (std::fabs(t0 + (double)s * dt - sa[j]) > 1e-9 * std::max(1.0, std::fabs(sa[j]))) return false;
    }
    if (j > 0 && s <= out[j - 1]) return false;
    out[j] = s;
  }
  return true;
}

// Save codes of a fixed-step Tsit5 run (tsit5.cuh::tsit5_save_coded): for each
// τ_j > t0, (s << 1) | interp with s the first step whose end tn(s) =
// (T)(t0 + s·dt) (tf for the last step) satisfies τ_j ≤ tn(s), interp = τ_j ≠
// tn(s). Host arithmetic mirrors the kernel's (IEEE, no contraction: the host
// side is compiled with -ffp-contract=off).
template <class T>
void fixed_save_codes(double t0, double tf, double dt, int64_t nsteps, const std::vector<T>& tau,
                      std::vector<int64_t>& code) {
  auto tn = [&](int64_t st) -> T {
    if (st >= nsteps) return (T)tf;
    const double prod = (double)st * dt;
    return (T)(t0 + prod);
  };
  code.assign(tau.size(), 0);
  for (size_t j = 0; j < tau.size(); ++j) {
    if (tau[j] <= (T)t0) continue;                       // saved at init
    int64_t st = (int64_t)std::ceil(((double)tau[j] - t0) / dt);
    st = std::min<int64_t>(std::max<int64_t>(st, 1), nsteps);
    while (st > 1 && tau[j] <= tn(st - 1)) --st;
    while (st < nsteps && tau[j] > tn(st)) ++st;
    code[j] = (st << 1) | (tau[j] == tn(st) ? 0 : 1);
  }
}

template <class T>
ens_status solve_impl(int model, int alg, int64_t N, int64_t ld, const void* u0, const void* p, double t0,
                      double tf, double dt, const ens_options* opt, const ens_output* out, int n,
                      cudaStream_t s, bool stage_ws) {
  const Layout L = layout(n, alg, sizeof(T) == 4 ? ENS_F32 : ENS_F64, N, opt);
  char* ws = (char*)out->workspace;
  Args<T> a{};
  a.N = N; a.ld = ld; a.ldo = opt->out_ld > 0 ? opt->out_ld : ld;
  a.u0 = (const T*)u0; a.p = (const T*)p; a.p_broadcast = opt->p_broadcast;
  a.t0d = t0; a.tfd = tf; a.dtd = dt;
  a.t0 = (T)t0; a.tf = (T)tf;
  int64_t nsteps; double hl;
  fixed_grid(t0, tf, dt, &nsteps, &hl);
  a.nsteps = nsteps; a.h_last = (T)hl;
  a.dt0 = opt->adaptive ? (T)std::min(dt, tf - t0) : (T)dt;
  a.abstol = (T)opt->abstol; a.reltol = (T)opt->reltol;
  // attempts = n_accept + n_reject (int32 counters), so a cap above INT32_MAX is unreachable
  a.max_steps = (int32_t)std::min<int64_t>(opt->max_steps > 0 ? opt->max_steps : 1000000, INT32_MAX);
  a.k = opt->n_saveat;
  a.tau = (const T*)(ws + L.tau);
  a.save_step = (const int64_t*)(ws + L.save_step);
  a.u_out = (T*)out->u_out; a.retcode = out->retcode; a.nacc = out->n_accept; a.nrej = out->n_reject;
  a.seed = opt->seed; a.rk = philox_round_keys(opt->seed); a.index_offset = opt->index_offset; a.chunk_len = opt->chunk_len;
  a.chunk_stride = opt->chunk_stride;
  a.partial = (double*)(ws + L.partial);
  a.counter = (unsigned long long*)(ws + L.counter);
  std::vector<int64_t> tsit_codes;   // fixed-step save codes (Tsit5: every chunk needs save_grid_only)
  if (coded_saves(alg, opt) && a.k > 0) {
    std::vector<T> tau(a.k);
    for (int j = 0; j < a.k; ++j) tau[j] = (T)opt->saveat[j];
    fixed_save_codes<T>(t0, tf, dt, nsteps, tau, tsit_codes);
    a.save_grid_only = std::all_of(tsit_codes.begin(), tsit_codes.end(), [](int64_t c) { return (c & 1) == 0; });
  }
  if (stage_ws) {
    if (a.k > 0) {
      std::vector<T> tau(a.k);
      for (int j = 0; j < a.k; ++j) tau[j] = (T)opt->saveat[j];
      if (cudaMemcpyAsync(ws + L.tau, tau.data(), sizeof(T) * a.k, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return ENS_E_CUDA;
      if (grid_saves(alg, opt)) {
        std::vector<int64_t> st;
        if (!em_save_steps(t0, tf, dt, opt->saveat, a.k, st)) return ENS_E_BAD_SAVEAT;
        if (cudaMemcpyAsync(ws + L.save_step, st.data(), 8 * a.k, cudaMemcpyHostToDevice, s) != cudaSuccess)
          return ENS_E_CUDA;
      } else if (coded_saves(alg, opt)) {
        if (cudaMemcpyAsync(ws + L.save_step, tsit_codes.data(), 8 * a.k, cudaMemcpyHostToDevice, s) != cudaSuccess)
          return ENS_E_CUDA;
      }
    }
  }
  if (opt->adaptive && opt->refill) {
    if (cudaMemsetAsync(ws + L.counter, 0, 8, s) != cudaSuccess) return ENS_E_CUDA;
  }
  ens_status st = dispatch<T>(model, alg, a, opt, s);
  if (st != ENS_OK) return st;
  if (opt->want_stats) {
    const bool fused = fused_stats(alg, opt);
    if (!is_sde_alg(alg) && !fused) {
      const dim3 g((unsigned)L.nparts, (unsigned)std::min(L.rows, kMaxGridY));
      stats_partial_kernel<T><<<g, kBlock, 0, s>>>((const T*)out->u_out, N, a.ldo, kStatsChunk, a.partial, L.rows);
    }
    // EM: one partial per block; fused Tsit5: one per warp (two trajectories per lane in fp32)
    const int64_t nparts = is_sde_alg(alg) ? (int64_t)grid_for(N).x
                           : fused ? cdiv(N, 32 * (sizeof(T) == 4 ? 2 : 1)) : L.nparts;
    if (nparts > 4 * 256 * kFold) {   // many partials (fused per-warp stats): fold in parallel first
      double* p2 = (double*)(ws + L.partial2);
      const int64_t nblk = cdiv(nparts, 256 * kFold);
      stats_fold_kernel<<<dim3((unsigned)nblk, (unsigned)std::min(L.rows, kMaxGridY)), 256, 0, s>>>(a.partial, nparts,
                                                                                                   p2, L.rows);
      stats_merge_kernel<<<L.rows, 256, 0, s>>>(p2, (int)nblk, out->stats);
    } else {
      stats_merge_kernel<<<L.rows, 256, 0, s>>>(a.partial, (int)nparts, out->stats);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return ENS_E_CUDA;
  }
  return ENS_OK;
}

}  // namespace

// =============================================================== C ABI =====
extern "C" {

ens_status ens_model_dims(ens_model model, int32_t* n, int32_t* m, int32_t* nw) {
  int a, b, c;
  if (!model_dims(model, &a, &b, &c)) return ENS_E_INVALID_ARG;
  if (n) *n = a;
  if (m) *m = b;
  if (nw) *nw = c;
  return ENS_OK;
}

size_t ens_workspace_bytes(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N, const ens_options* opt) {
  int n, m, nw;
  if (!model_dims(model, &n, &m, &nw)) return 0;
  return layout(n, alg, dtype, N, opt).total;
}

ens_status ensemble_solve(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N, const void* u0, const void* p,
                          double t0, double tf, double dt, const ens_options* opt, ens_output* out, void* stream) {
  int n = 0;
  ens_status st = validate(model, alg, dtype, N, t0, tf, dt, opt, &n);
  if (st != ENS_OK) return st;
  if (!out || !u0 || !p) return ENS_E_INVALID_ARG;
  if (!out->u_out && !(is_sde_alg(alg) && opt->want_stats)) return ENS_E_INVALID_ARG;
  if (opt->want_stats && !out->stats) return ENS_E_INVALID_ARG;
  if (grid_saves(alg, opt) && opt->n_saveat > 0) {
    std::vector<int64_t> tmp;
    if (!em_save_steps(t0, tf, dt, opt->saveat, opt->n_saveat, tmp)) return ENS_E_BAD_SAVEAT;
  }
  if (!out->workspace || out->workspace_bytes < ens_workspace_bytes(model, alg, dtype, N, opt)) return ENS_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == ENS_F32) return solve_impl<float>(model, alg, N, N, u0, p, t0, tf, dt, opt, out, n, s, true);
  return solve_impl<double>(model, alg, N, N, u0, p, t0, tf, dt, opt, out, n, s, true);
}

ens_status ensemble_solve_host(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N, const void* u0_host,
                               const void* p_host, double t0, double tf, double dt, const ens_options* opt,
                               void* d_u0, void* d_p, void* d_u_out, int32_t* d_retcode, void* u_out_host,
                               int32_t* retcode_host, void* workspace, size_t workspace_bytes, int32_t n_chunks,
                               void* stream) {
  int n = 0, m = 0, nw = 0;
  ens_status st = validate(model, alg, dtype, N, t0, tf, dt, opt, &n);
  if (st != ENS_OK) return st;
  if (opt->want_stats || opt->out_ld != 0) return ENS_E_UNSUPPORTED;
  if (!u0_host || !p_host || !d_u0 || !d_p || !d_u_out || !u_out_host) return ENS_E_INVALID_ARG;
  const int64_t C = std::max<int64_t>(1, std::min<int64_t>(n_chunks, N));
  // Philox counters key on the global trajectory index (DESIGN R10): each chunk
  // shifts index_offset by its start; a block-cyclic map cannot be split that way.
  if (is_sde_alg(alg) && opt->chunk_len > 0 && C > 1) return ENS_E_UNSUPPORTED;
  if (grid_saves(alg, opt) && opt->n_saveat > 0) {
    std::vector<int64_t> tmp;
    if (!em_save_steps(t0, tf, dt, opt->saveat, opt->n_saveat, tmp)) return ENS_E_BAD_SAVEAT;
  }
  if (!workspace || workspace_bytes < ens_workspace_bytes(model, alg, dtype, N, opt)) return ENS_E_WORKSPACE;
  model_dims(model, &n, &m, &nw);
  const size_t ts = dtype == ENS_F32 ? 4 : 8;
  const int kk = std::max(1, opt->n_saveat);
  cudaStream_t s = (cudaStream_t)stream;
  cudaStream_t sh = nullptr, sd = nullptr, s2 = nullptr;
  if (cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking) != cudaSuccess) return ENS_E_CUDA;
  if (cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking) != cudaSuccess) { cudaStreamDestroy(sh); return ENS_E_CUDA; }
  // Odd chunks solve on a second compute stream, so a chunk's kernel fills the
  // SMs its predecessor's last partial wave leaves idle (one stream would
  // serialise the launches and expose every chunk's tail). Not with refill: its
  // per-launch queue counter lives in the shared workspace.
  const bool dual = C > 1 && !(opt->adaptive && opt->refill);
  if (dual && cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess) {
    cudaStreamDestroy(sh); cudaStreamDestroy(sd); return ENS_E_CUDA;
  }
  cudaEvent_t staged = nullptr, s2_done = nullptr;
  if (dual) {
    cudaEventCreateWithFlags(&staged, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&s2_done, cudaEventDisableTiming);
  }
  std::vector<cudaEvent_t> ev_in(C), ev_out(C);
  for (int64_t c = 0; c < C; ++c) {
    cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out[c], cudaEventDisableTiming);
  }
  ens_output out{};
  out.workspace = workspace; out.workspace_bytes = workspace_bytes;
  bool ok = true;
  // stage saveat once (stream-ordered on s)
  cudaEvent_t start;
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventRecord(start, s);
  cudaStreamWaitEvent(sh, start, 0);
  // Chunk sizes: with 8+ chunks the first and last three ramp (weights 1, 2, 4 against 8 for the
  // middle ones) so the copy-in of the first chunk and the copy-out of the last — the parts of the
  // pipeline no compute overlaps — are small.
  std::vector<int64_t> wgt(C, 8);
  if (C >= 8 && N >= 1024 * 8 * C)   // (large N only: every chunk stays non-empty)
    for (int j = 0; j < 3; ++j) wgt[j] = wgt[C - 1 - j] = (int64_t)1 << j;
  int64_t wsum = 0;
  for (int64_t c = 0; c < C; ++c) wsum += wgt[c];
  std::vector<int64_t> bound(C + 1, 0);
  for (int64_t c = 0, acc = 0; c < C; ++c) {
    acc += wgt[c];
    bound[c + 1] = (int64_t)((__int128)N * acc / wsum);
  }
  int64_t lo = 0;
  for (int64_t c = 0; c < C && ok; ++c) {
    const int64_t len = bound[c + 1] - bound[c];
    // H2D of chunk c (component rows are strided by N in the SoA layout)
    ok &= cudaMemcpy2DAsync((char*)d_u0 + lo * ts, N * ts, (const char*)u0_host + lo * ts, N * ts, len * ts, n,
                            cudaMemcpyHostToDevice, sh) == cudaSuccess;
    if (opt->p_broadcast) {
      if (c == 0) ok &= cudaMemcpyAsync(d_p, p_host, m * ts, cudaMemcpyHostToDevice, sh) == cudaSuccess;
    } else {
      ok &= cudaMemcpy2DAsync((char*)d_p + lo * ts, N * ts, (const char*)p_host + lo * ts, N * ts, len * ts, m,
                              cudaMemcpyHostToDevice, sh) == cudaSuccess;
    }
    cudaEventRecord(ev_in[c], sh);
    cudaStream_t cs = (dual && (c & 1)) ? s2 : s;
    if (dual && c == 1) cudaStreamWaitEvent(s2, staged, 0);   // after chunk 0 staged saveat into the workspace
    cudaStreamWaitEvent(cs, ev_in[c], 0);
    out.u_out = (char*)d_u_out + lo * ts;
    out.retcode = d_retcode ? d_retcode + lo : nullptr;
    ens_options o = *opt;
    if (o.chunk_len == 0) o.index_offset = opt->index_offset + lo;
    const void* pp = opt->p_broadcast ? d_p : (const void*)((const char*)d_p + lo * ts);
    if (dtype == ENS_F32)
      st = solve_impl<float>(model, alg, len, N, (const char*)d_u0 + lo * ts, pp, t0, tf, dt, &o, &out, n, cs, c == 0);
    else
      st = solve_impl<double>(model, alg, len, N, (const char*)d_u0 + lo * ts, pp, t0, tf, dt, &o, &out, n, cs, c == 0);
    if (st != ENS_OK) { ok = false; break; }
    if (dual && c == 0) cudaEventRecord(staged, s);
    cudaEventRecord(ev_out[c], cs);
    cudaStreamWaitEvent(sd, ev_out[c], 0);
    ok &= cudaMemcpy2DAsync((char*)u_out_host + lo * ts, N * ts, (const char*)d_u_out + lo * ts, N * ts, len * ts,
                            (size_t)kk * n, cudaMemcpyDeviceToHost, sd) == cudaSuccess;
    if (retcode_host && d_retcode)
      ok &= cudaMemcpyAsync(retcode_host + lo, d_retcode + lo, len * 4, cudaMemcpyDeviceToHost, sd) == cudaSuccess;
    lo += len;
  }
  if (dual) {                                // the caller's stream orders after every chunk
    cudaEventRecord(s2_done, s2);
    cudaStreamWaitEvent(s, s2_done, 0);
  }
  ok &= cudaStreamSynchronize(sd) == cudaSuccess;
  ok &= cudaStreamSynchronize(s) == cudaSuccess;
  cudaStreamSynchronize(sh);
  if (dual) {
    cudaEventDestroy(staged);
    cudaEventDestroy(s2_done);
    cudaStreamDestroy(s2);
  }
  for (int64_t c = 0; c < C; ++c) { cudaEventDestroy(ev_in[c]); cudaEventDestroy(ev_out[c]); }
  cudaEventDestroy(start);
  cudaStreamDestroy(sh);
  cudaStreamDestroy(sd);
  if (st != ENS_OK) return st;
  return ok ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_generate_inputs(ens_model model, ens_dtype dtype, ens_recipe recipe, uint64_t input_seed, int64_t N,
                               int64_t N_total, const ens_options* opt, void* u0, void* p, void* stream) {
  InputSpec sp{};
  int nw;
  if (!model_dims(model, &sp.n, &sp.m, &nw) || N < 1 || !u0 || !p) return ENS_E_INVALID_ARG;
  if (recipe < ENS_RECIPE_RANDOM10 || recipe > ENS_RECIPE_GRID) return ENS_E_INVALID_ARG;
  if (recipe == ENS_RECIPE_RHO_SWEEP && model != ENS_LORENZ) return ENS_E_UNSUPPORTED;
  if ((recipe == ENS_RECIPE_GRID) != (model == ENS_CRN)) return ENS_E_UNSUPPORTED;
  // p̄ and ū0 of DESIGN §6 (same table as synth/inputs.py); CRN: Table-5 ranges (lo, hi)
  static const double PB[7][4] = {{10.0, 28.0, 8.0 / 3.0, 0}, {0.04, 3e7, 1e4, 0}, {10.0, 28.0, 8.0 / 3.0, 0.1},
                                  {10.0, 28.0, 8.0 / 3.0, 0.1}, {1.5, 0.01, 0, 0}, {1.0, 0, 0, 0}, {1.0, 0, 0, 0}};
  static const double UB[7][3] = {{1, 0, 0}, {1, 0, 0}, {1, 0, 0}, {1, 0, 0}, {0.1, 0.1, 0.1}, {1, 0, 0}, {1, 0, 0}};
  static const double CRN_LO[6] = {0.1, 0.1, 0.1, 0.01, 2.0, 0.001}, CRN_HI[6] = {100.0, 100.0, 100.0, 0.2, 4.0, 0.1};
  // stiff suite: rate constants and initial states as printed
  static const double OREGO_P[3] = {77.27, 8.375e-6, 0.161}, OREGO_U[3] = {1.0, 2.0, 3.0};
  static const double HIRES_P[12] = {1.71, 0.43, 8.32, 0.0007, 8.75, 10.03, 0.035, 1.12, 1.745, 280.0, 0.69, 1.81};
  static const double HIRES_U[8] = {1.0, 0, 0, 0, 0, 0, 0, 0.0057};
  static const double POLLU_P[25] = {0.35, 26.6, 12300.0, 0.00086, 0.00082, 15000.0, 0.00013, 24000.0, 16500.0,
                                     9000.0, 0.022, 12000.0, 1.88, 16300.0, 4.8e6, 0.00035, 0.0175, 1.0e8, 4.44e11,
                                     1240.0, 2.1, 5.78, 0.0474, 1780.0, 3.12};
  static const double POLLU_U[20] = {0.0, 0.2, 0.0, 0.04, 0.0, 0.0, 0.1, 0.3, 0.017, 0.0,
                                     0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.007, 0.0, 0.0, 0.0};
  if (model == ENS_BALL) {   // g = 9.8, e = 0.85 (varies, R18); dropped from x = 50 at rest
    sp.pbar[0] = 9.8; sp.pbar[1] = 0.85;
    sp.ubar[0] = 50.0; sp.ubar[1] = 0.0;
  } else if (model >= ENS_OREGO) {
    const double* pb = model == ENS_OREGO ? OREGO_P : model == ENS_HIRES ? HIRES_P : POLLU_P;
    const double* ub = model == ENS_OREGO ? OREGO_U : model == ENS_HIRES ? HIRES_U : POLLU_U;
    for (int j = 0; j < sp.m; ++j) sp.pbar[j] = pb[j];
    for (int j = 0; j < sp.n; ++j) sp.ubar[j] = ub[j];
  } else
  if (model == ENS_CRN) {
    for (int j = 0; j < 6; ++j) { sp.lo[j] = CRN_LO[j]; sp.hi[j] = CRN_HI[j]; }
    const int64_t nt = N_total > 0 ? N_total : N;
    int64_t L = 2;
    while (true) {                       // smallest L >= 2 with L^6 >= N_total
      int64_t pw = 1;
      for (int j = 0; j < 6; ++j) pw *= L;
      if (pw >= nt) break;
      ++L;
    }
    sp.levels = L;
  } else {
    for (int j = 0; j < 4; ++j) sp.pbar[j] = PB[model][j];
    for (int j = 0; j < 3; ++j) sp.ubar[j] = UB[model][j];
  }
  sp.recipe = recipe;
  sp.n_total = (double)(N_total > 0 ? N_total : N);
  const int64_t off = opt ? opt->index_offset : 0, cl = opt ? opt->chunk_len : 0, cs = opt ? opt->chunk_stride : 0;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 g((unsigned)cdiv(N, kBlock));
  if (dtype == ENS_F32) generate_inputs_kernel<float><<<g, kBlock, 0, s>>>(sp, input_seed, N, off, cl, cs, (float*)u0, (float*)p);
  else generate_inputs_kernel<double><<<g, kBlock, 0, s>>>(sp, input_seed, N, off, cl, cs, (double*)u0, (double*)p);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

size_t ens_stats_workspace_bytes(int64_t N, int32_t rows) {
  if (N < 1 || rows < 1) return 0;
  return align256((size_t)rows * (size_t)cdiv(N, kStatsChunk) * 3 * 8) + 256;
}

ens_status ens_ensemble_stats(ens_dtype dtype, const void* x, int64_t N, int64_t ld, int32_t rows, double* stats,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (!x || !stats || N < 1 || ld < N || rows < 1 || (dtype != ENS_F32 && dtype != ENS_F64)) return ENS_E_INVALID_ARG;
  if (!workspace || workspace_bytes < ens_stats_workspace_bytes(N, rows)) return ENS_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nparts = cdiv(N, kStatsChunk);
  const dim3 g((unsigned)nparts, (unsigned)std::min(rows, kMaxGridY));
  double* part = (double*)workspace;
  if (dtype == ENS_F32)
    stats_partial_kernel<float><<<g, kBlock, 0, s>>>((const float*)x, N, ld, kStatsChunk, part, rows);
  else stats_partial_kernel<double><<<g, kBlock, 0, s>>>((const double*)x, N, ld, kStatsChunk, part, rows);
  stats_merge_kernel<<<rows, 256, 0, s>>>(part, (int)nparts, stats);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_stats_finalize(const double* stats, int32_t k, int32_t n, double* mean, double* var, void* stream) {
  if (!stats || !mean || !var || n < 1 || k < 0) return ENS_E_INVALID_ARG;
  const int rows = std::max(1, k) * n;
  stats_finalize_kernel<<<cdiv(rows, 128), 128, 0, (cudaStream_t)stream>>>(stats, rows, mean, var);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_stats_merge(const double* gathered, int32_t R, int32_t k, int32_t n, double* merged, void* stream) {
  if (!gathered || !merged || R < 1 || n < 1 || k < 0) return ENS_E_INVALID_ARG;
  const int rows = std::max(1, k) * n;
  stats_rank_merge_kernel<<<cdiv(rows, 128), 128, 0, (cudaStream_t)stream>>>(gathered, R, rows, merged);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_sde_noise(ens_dtype dtype, uint64_t seed, int64_t N, int64_t step0, int64_t nsteps, int32_t nw,
                         const ens_options* opt, uint32_t* words, void* z, void* stream) {
  if (N < 1 || nsteps < 0 || step0 < 0 || (dtype != ENS_F32 && dtype != ENS_F64)) return ENS_E_INVALID_ARG;
  if (nw != 3 && nw != 8) return ENS_E_UNSUPPORTED;
  const int64_t off = opt ? opt->index_offset : 0, cl = opt ? opt->chunk_len : 0, cs = opt ? opt->chunk_stride : 0;
  const dim3 g((unsigned)cdiv(N, kBlock));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == ENS_F32) {
    if (nw == 3) sde_noise_kernel<float, 3><<<g, kBlock, 0, s>>>(philox_round_keys(seed), N, step0, nsteps, off, cl, cs, words, (float*)z);
    else sde_noise_kernel<float, 8><<<g, kBlock, 0, s>>>(philox_round_keys(seed), N, step0, nsteps, off, cl, cs, words, (float*)z);
  } else {
    if (nw == 3) sde_noise_kernel<double, 3><<<g, kBlock, 0, s>>>(philox_round_keys(seed), N, step0, nsteps, off, cl, cs, words, (double*)z);
    else sde_noise_kernel<double, 8><<<g, kBlock, 0, s>>>(philox_round_keys(seed), N, step0, nsteps, off, cl, cs, words, (double*)z);
  }
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int64_t N, void* stream) {
  if (!ctr || !key || !out || N < 1) return ENS_E_INVALID_ARG;
  philox_kernel<<<(unsigned)cdiv(N, kBlock), kBlock, 0, (cudaStream_t)stream>>>(ctr, key, out, N);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

ens_status ens_check_fast_paths(unsigned long long* mismatches, void* stream) {
  if (!mismatches) return ENS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(mismatches, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess) return ENS_E_CUDA;
  // m ∈ [(float)√½, 2·(float)√½): every m that L(x) forms (frexp mantissa, doubled below √½)
  log2_quot_check_kernel<<<4 * sm_count(), kBlock, 0, s>>>(0x3F3504F3u, 0x3FB504F3u, mismatches);
  // x ∈ [1e-7, 64): every Box–Muller radicand −2 ln U of the fp32 uniforms
  bm_sqrt_check_kernel<<<8 * sm_count(), kBlock, 0, s>>>(0x33D6BF95u, 0x42800000u, mismatches + 1);
  return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA;
}

const char* ens_status_string(ens_status s) {
  switch (s) {
    case ENS_OK: return "ok";
    case ENS_E_INVALID_ARG: return "invalid argument";
    case ENS_E_ALG_MISMATCH: return "algorithm does not match the model kind (ODE vs SDE)";
    case ENS_E_ADAPTIVE_UNSUPPORTED: return "adaptive stepping is not supported for this algorithm";
    case ENS_E_BAD_TOLERANCE: return "bad tolerance (abstol must be > 0, reltol >= 0)";
    case ENS_E_BAD_TSPAN: return "bad time span or step (need t0 < tf, dt > 0, all finite)";
    case ENS_E_BAD_SAVEAT: return "bad saveat (must be strictly increasing in [t0, tf]; EM: on the step grid)";
    case ENS_E_WORKSPACE: return "workspace missing or too small";
    case ENS_E_UNSUPPORTED: return "unsupported combination";
    case ENS_E_CUDA: return "CUDA error";
  }
  return "unknown status";
}

const char* ens_version(void) { return "ens-b200 0.2 (sm_100a)"; }

}  // extern "C"
