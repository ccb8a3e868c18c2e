// tsit5.cuh — per-thread Tsit5 5(4) integrator for sm_100a.
//
// One trajectory per lane (the paper's EnsembleGPUKernel, Listing 1
// P:287-307); the fixed-step fp32 kernel carries TWO trajectories per thread
// in packed f2 lanes (FFMA2/FADD2/FMUL2), bit-identical per trajectory. State,
// the seven stage vectors, the error estimate and the controller live in
// registers ("stack allocate all intermediates").
//
// Stage sums (DESIGN R1, §4): y_i = u + Σ_{l<i} (h·a_il) k_l, evaluated
//     y = u; y = fma(h·a_il, k_l, y)  (l = 1..i−1)
// with the products h·a_il rounded to T: i−1 FMAs per component and stage.
// Fixed-step runs take the 21 products from kernel parameters (computed once
// on the host, uniform registers in SASS); adaptive runs form them per step.
#pragma once
#include "common.cuh"
#include "models.cuh"
#include "stats.cuh"
#include "vec2.cuh"

namespace ens {

// Tsitouras (2011) coefficients, as published (Tsit5). Double literals,
// converted to T once (DESIGN R7).
__host__ __device__ constexpr double ts_a(int i, int j) {
  constexpr double A[7][7] = {
      {0, 0, 0, 0, 0, 0, 0},
      {0.161, 0, 0, 0, 0, 0, 0},
      {-0.008480655492356989, 0.335480655492357, 0, 0, 0, 0, 0},
      {2.897153057105493, -6.359448489975075, 4.3622954328695815, 0, 0, 0, 0},
      {5.325864828439257, -11.748883564062828, 7.4955393428898365, -0.09249506636175525, 0, 0, 0},
      {5.86145544294642, -12.92096931784711, 8.159367898576159, -0.071584973281401, -0.028269050394068383, 0, 0},
      {0.09646076681806523, 0.01, 0.4798896504144996, 1.379008574103742, -3.290069515436081, 2.324710524099774,
       0}};
  return A[i][j];
}
__host__ __device__ constexpr double ts_c(int i) {
  constexpr double C[7] = {0.0, 0.161, 0.327, 0.9, 0.9800255409045097, 1.0, 1.0};
  return C[i];
}
// b̃ = b − b̂ (embedded order-4 difference weights)
__host__ __device__ constexpr double ts_bt(int i) {
  constexpr double B[7] = {-0.00178001105222577714, -0.0008164344596567469, 0.007880878010261995,
                           -0.1447110071732629,     0.5823571654525552,     -0.45808210592918697,
                           0.015151515151515152};
  return B[i];
}
// free 4th-order interpolant: b_1(θ) = θ(r11+θ(r12+θ(r13+θ r14))), b_i(θ) = θ²(r_i2+θ(r_i3+θ r_i4))
__host__ __device__ constexpr double ts_r(int i, int j) {
  constexpr double R[7][4] = {{1.0, -2.763706197274826, 2.9132554618219126, -1.0530884977290216},
                              {0.0, 0.13169999999999998, -0.2234, 0.1017},
                              {0.0, 3.9302962368947516, -5.941033872131505, 2.490627285651253},
                              {0.0, -12.411077166933676, 30.33818863028232, -16.548102889244902},
                              {0.0, 37.50931341651104, -88.1789048947664, 47.37952196281928},
                              {0.0, -27.896526289197286, 65.09189467479366, -34.87065786149661},
                              {0.0, 1.5, -4.0, 2.5}};
  return R[i][j];
}
constexpr int kEventPts = 10;   // event-condition samples per accepted step (DESIGN R18)

// (i, l), 1 ≤ i ≤ 6, l < i  →  0..20
__host__ __device__ constexpr int ts_idx(int i, int l) { return i * (i - 1) / 2 + l; }

// Step-scaled coefficients h·a_il for the fixed step dt (h) and the last step (hl).
// C = float, double, or float2 (the same float product broadcast to both lanes).
template <class C> struct TsitCoef { C h[21]; C hl[21]; };
template <class V> struct CoefOf { using C = V; };
template <> struct CoefOf<f2> { using C = float2; };
__device__ __forceinline__ float coef_to(float c, float*) { return c; }
__device__ __forceinline__ double coef_to(double c, double*) { return c; }
__device__ __forceinline__ f2 coef_to(float2 c, f2*) { return f2(c); }

template <class V, class C> struct HaParam {      // coefficients read from kernel parameters
  const C* p;
  __device__ __forceinline__ V operator()(int i, int l) const { return coef_to(p[ts_idx(i, l)], (V*)nullptr); }
};
template <class V> struct HaReg {                  // coefficients formed in registers for this step
  V v[21];
  __device__ __forceinline__ explicit HaReg(V h) {
#pragma unroll
    for (int i = 1; i < 7; ++i)
#pragma unroll
      for (int l = 0; l < i; ++l) v[ts_idx(i, l)] = h * V(ts_a(i, l));
  }
  __device__ __forceinline__ V operator()(int i, int l) const { return v[ts_idx(i, l)]; }
};

// Stages 2..7 from (t, u, K[0] = f(u)): fills K[1..6] and y = u_{n+1} (= y_7, FSAL).
template <class M, class V, class HA>
__device__ __forceinline__ void tsit5_stages(const V (&par)[M::m], V t, V h, const HA& ha, const V (&u)[M::n],
                                             V (&K)[7][M::n], V (&y)[M::n]) {
  constexpr int n = M::n;
#pragma unroll
  for (int i = 1; i < 7; ++i) {
#pragma unroll
    for (int j = 0; j < n; ++j) {
      V acc = u[j];
#pragma unroll
      for (int l = 0; l < i; ++l) acc = fmaT(ha(i, l), K[l][j], acc);
      y[j] = acc;
    }
    M::f(y, par, t + V(ts_c(i)) * h, K[i]);
  }
}

// E = h Σ b̃_i k_i
template <int n, class T>
__device__ __forceinline__ void tsit5_error(T h, const T (&K)[7][n], T (&E)[n]) {
#pragma unroll
  for (int j = 0; j < n; ++j) {
    T e = T(ts_bt(0)) * K[0][j];
#pragma unroll
    for (int l = 1; l < 7; ++l) e = fmaT(T(ts_bt(l)), K[l][j], e);
    E[j] = h * e;
  }
}

// u(t + θh) = u + h Σ b_i(θ) k_i
template <int n, class V>
__device__ __forceinline__ void tsit5_interp(V theta, V h, const V (&u)[n], const V (&K)[7][n], V (&o)[n]) {
  V bt[7];
  bt[0] = fmaT(theta, fmaT(theta, fmaT(theta, V(ts_r(0, 3)), V(ts_r(0, 2))), V(ts_r(0, 1))), V(ts_r(0, 0))) * theta;
  const V th2 = theta * theta;
#pragma unroll
  for (int i = 1; i < 7; ++i) bt[i] = fmaT(theta, fmaT(theta, V(ts_r(i, 3)), V(ts_r(i, 2))), V(ts_r(i, 1))) * th2;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    V acc = bt[0] * K[0][j];
#pragma unroll
    for (int i = 1; i < 7; ++i) acc = fmaT(bt[i], K[i][j], acc);
    o[j] = fmaT(h, acc, u[j]);
  }
}

// ---------------------------------------------------- lane load / store --
template <class M, class V, class T>
__device__ __forceinline__ void load_lanes(const Args<T>& a, const int64_t (&idx)[LaneOf<V>::W], V (&u)[M::n],
                                           V (&par)[M::m]) {
  constexpr int W = LaneOf<V>::W;
#pragma unroll
  for (int c = 0; c < M::n; ++c) {
    T x[2];
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = __ldg(a.u0 + (size_t)c * a.ld + idx[w]);
    u[c] = make_lanes<V>(x[0], x[W - 1]);
  }
#pragma unroll
  for (int c = 0; c < M::m; ++c) {
    T x[2];
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = a.p_broadcast ? __ldg(a.p + c) : __ldg(a.p + (size_t)c * a.ld + idx[w]);
    par[c] = make_lanes<V>(x[0], x[W - 1]);
  }
}

template <int n, class V, class T>
__device__ __forceinline__ void store_lanes(const Args<T>& a, const int64_t (&idx)[LaneOf<V>::W],
                                            const bool (&live)[LaneOf<V>::W], int j, const V (&v)[n]) {
  if constexpr (LaneOf<V>::W == 2) {
    // a thread's two trajectories are neighbours in memory: one 8-byte store per
    // component (a warp writes 256 contiguous bytes) when both lanes are live and the
    // pair is 8-byte aligned (a lane that diverged at t0 keeps its u0 / NaN saves)
    if (live[0] && live[1] && (a.ldo % 2) == 0 && (reinterpret_cast<uintptr_t>(a.u_out) & 7) == 0) {
#pragma unroll
      for (int c = 0; c < n; ++c)
        *reinterpret_cast<float2*>(a.u_out + ((size_t)j * n + c) * a.ldo + idx[0]) = v[c].v;
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < LaneOf<V>::W; ++w)
    if (live[w]) {
#pragma unroll
      for (int c = 0; c < n; ++c) a.u_out[((size_t)j * n + c) * a.ldo + idx[w]] = lane(v[c], w);
    }
}

template <int n, class V>
__device__ __forceinline__ bool lane_finite(const V (&v)[n], int w) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < n; ++c) ok = ok && finiteT(lane(v[c], w));
  return ok;
}

// Save every τ_j ∈ (t, tn] of an accepted step [t, tn] (DESIGN R5). In
// fixed-step runs t, tn, h are shared by the lanes of a thread.
template <int n, class V, class T>
__device__ __forceinline__ void tsit5_save(const Args<T>& a, const int64_t (&idx)[LaneOf<V>::W],
                                           const bool (&live)[LaneOf<V>::W], int& js, T t, T tn, T h,
                                           const V (&u)[n], const V (&K)[7][n], const V (&un)[n]) {
  while (js < a.k) {
    const T tau = __ldg(a.tau + js);
    if (!(tau <= tn)) break;
    if (tau == tn) {
      store_lanes<n, V, T>(a, idx, live, js, un);
    } else {
      V o[n];
      tsit5_interp<n, V>(splat<V>((tau - t) / h), splat<V>(h), u, K, o);
      store_lanes<n, V, T>(a, idx, live, js, o);
    }
    ++js;
  }
}

// Fixed-step saves by precomputed step codes (host: fixed_save_codes in api.cu):
// save_step[j] = (s << 1) | interp, s = the 1-based step after which τ_j is
// stored — the first s with τ_j ≤ tn(s), tn(s) = (T)(t0 + s·dt) (tf for the
// last step), the same comparison the per-step scan made — and interp = 0 if
// τ_j == tn(s) exactly (store u_{s}) else 1 (interpolant at θ = (τ_j − t)/h).
// Steps without a save then cost one integer compare instead of a time
// computation and a τ load.
template <int n, class V, class T, bool INTERP>
__device__ __forceinline__ void tsit5_save_coded(const Args<T>& a, const int64_t (&idx)[LaneOf<V>::W],
                                                 const bool (&live)[LaneOf<V>::W], int& js, int64_t& next,
                                                 int64_t s, T h, const V (&u)[n], const V (&K)[7][n],
                                                 const V (&un)[n]) {
  while (js < a.k) {
    const int64_t code = __ldg(a.save_step + js);
    if ((code >> 1) != s + 1) { next = code >> 1; return; }
    if (INTERP && (code & 1)) {
      const T t = (T)(a.t0d + (double)s * a.dtd);
      V o[n];
      tsit5_interp<n, V>(splat<V>((__ldg(a.tau + js) - t) / h), splat<V>(h), u, K, o);
      store_lanes<n, V, T>(a, idx, live, js, o);
    } else {
      store_lanes<n, V, T>(a, idx, live, js, un);
    }
    ++js;
  }
  next = -1;
}

// Bulk (TMA-engine) stores of grid saves: every thread of a full block puts its
// values into a shared-memory row buffer; one thread then streams each
// component row — blockDim·W contiguous values — to global memory with
// cp.async.bulk (UBLKCP), double-buffered, so the save traffic leaves the SM as
// large asynchronous writes instead of per-thread stores in the step loop.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int n, class V, class T>
__device__ __forceinline__ void tsit5_save_bulk(const Args<T>& a, const bool (&live)[LaneOf<V>::W], int& js,
                                                int& nb, int64_t& next, int64_t s, const V (&un)[n], int64_t blk0,
                                                T* smem) {
  constexpr int W = LaneOf<V>::W;
  const int BW = blockDim.x * W;
  while (js < a.k) {
    const int64_t code = __ldg(a.save_step + js);
    if ((code >> 1) != s + 1) { next = code >> 1; return; }
    T* buf = smem + (size_t)(nb & 1) * n * BW;
    if (nb >= 2) {                            // this buffer was last read by the copies of save nb − 2
      if (threadIdx.x == 0) bulk_wait_read1();
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < n; ++c) {
      if constexpr (W == 2) {
        *reinterpret_cast<float2*>(buf + (size_t)c * BW + 2 * threadIdx.x) =
            make_float2(live[0] ? lane(un[c], 0) : nanT<float>(), live[1] ? lane(un[c], 1) : nanT<float>());
      } else {
        buf[(size_t)c * BW + threadIdx.x] = live[0] ? lane(un[c], 0) : nanT<T>();
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < n; ++c)
        bulk_s2g(a.u_out + ((size_t)js * n + c) * a.ldo + blk0, buf + (size_t)c * BW, (uint32_t)(BW * sizeof(T)));
      bulk_commit();
    }
    ++nb;
    ++js;
  }
  next = -1;
}

// ---------------------------------------------------------------- fixed dt --
// Fixed grid (DESIGN R3): nsteps steps of dt, the last of h_last. No error
// estimate. Divergence is checked on f(u0) and the final state (DESIGN R6).
// V = float2-pair (two trajectories per thread), float or double.
// SAVE: 0 = final state only; 1 = saveat with interpolation between grid
// points; 2 = every save point on the step grid (no interpolant, so the stage
// vectors are dead after each step: fewer registers, coefficients stay in
// uniform registers); 3 = as 2, full blocks stream their saves through shared
// memory with bulk copies (dynamic shared memory 2·n·blockDim·W·sizeof(T);
// the host checks the 16-byte alignment of every row).
// Epilogue of the STATS instances, out of line so that it does not take part in
// the register allocation of the step loop. Arguments are scalars and a small
// aggregate by value: a reference to the kernel's Args (or to register arrays)
// would force a per-thread copy into local memory (352 B, i.e. 1.7 GB of DRAM
// writes per N = 10^7 launch).
template <int n, int W, class T> struct FinalPack {
  T y[n][W];
  int64_t idx[W];
  bool live[W];
};
template <int n, int W, class T>
__device__ __noinline__ void fused_final_stats(int64_t N, int64_t ld, const T* __restrict__ u0,
                                               double* __restrict__ partial, int64_t i0, const FinalPack<n, W, T> fp) {
  const int64_t nparts = cdiv_dev(N, 32 * W);
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
  for (int c = 0; c < n; ++c) {
    double x[W];
    bool use[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const bool valid = i0 + w < N, div0 = valid && !fp.live[w];   // live is cleared only by a t0 divergence
      x[w] = div0 ? (double)__ldg(u0 + (size_t)c * ld + fp.idx[w]) : (double)fp.y[c][w];
      use[w] = valid && isfinite(x[w]);
    }
    warp_stats_partial<W>(use, x, partial + ((size_t)c * nparts + wg) * 3);
  }
}

// STATS (final state only): fused ensemble statistics of the stored final
// states — one (count, mean, M2) partial per warp into a.partial
// [n][cdiv(N, 32·W)][3], merged by stats_merge_kernel — so the states are not
// read back (on a multi-GPU run they may live in another GPU's memory).
template <class M, class V, int SAVE, bool STATS = false>
__global__ void __launch_bounds__(256)
    tsit5_fixed_kernel(const Args<typename LaneOf<V>::T> a, const TsitCoef<typename CoefOf<V>::C> cf) {
  static_assert(!STATS || SAVE == 0, "fused statistics are for final-state solves");
  using T = typename LaneOf<V>::T;
  using C = typename CoefOf<V>::C;
  constexpr int n = M::n, W = LaneOf<V>::W;
  extern __shared__ __align__(16) unsigned char ens_fixed_smem[];
  const int64_t blk0 = (int64_t)blockIdx.x * blockDim.x * W;
  // bulk saves need every thread of the block at every barrier: full blocks only
  const bool bulk = (SAVE == 3) && (blk0 + (int64_t)blockDim.x * W <= a.N);
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
  if (STATS) {   // the warp reduction needs every lane of a warp with any trajectory
    if (((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * W >= a.N) return;
  } else if (i0 >= a.N) {
    return;
  }
  int64_t idx[W];
  bool live[W];
#pragma unroll
  for (int w = 0; w < W; ++w) { idx[w] = min(i0 + w, a.N - 1); live[w] = (i0 + w < a.N); }
  V u[n], par[M::m], K[7][n], y[n];
  load_lanes<M, V, T>(a, idx, u, par);
  M::f(u, par, splat<V>(a.t0), K[0]);
  int js = 0;
  if (SAVE) {
    while (js < a.k && __ldg(a.tau + js) <= a.t0) { store_lanes<n, V, T>(a, idx, live, js, u); ++js; }
  }
  const int64_t steps = a.nsteps;
  // a lane whose f(u0) is non-finite is finished now (Diverged, no step taken)
#pragma unroll
  for (int w = 0; w < W; ++w) {
    if (live[w] && !lane_finite<n, V>(K[0], w)) {
      for (int j = js; j < (SAVE ? a.k : 1); ++j)
#pragma unroll
        for (int c = 0; c < n; ++c)
          a.u_out[((size_t)j * n + c) * a.ldo + idx[w]] = SAVE ? nanT<T>() : lane(u[c], w);
      if (a.retcode) a.retcode[idx[w]] = RET_DIVERGED;
      if (a.nacc) a.nacc[idx[w]] = 0;
      if (a.nrej) a.nrej[idx[w]] = 0;
      live[w] = false;
    }
  }
  bool any = false;
#pragma unroll
  for (int w = 0; w < W; ++w) any = any || live[w];
  // (in a bulk block a finished thread stays for the barriers, saving NaN; with
  //  STATS it stays for the warp reduction)
  if (!any && !bulk && !STATS) return;
  int nb = 0;                   // bulk saves issued by this block
  const V hdt = splat<V>(a.dt0);
  const HaParam<V, C> ha{cf.h};
  int64_t next = -1;   // step after which the next save falls (SAVE)
  if (SAVE && js < a.k) next = __ldg(a.save_step + js) >> 1;
  // all steps but the last: constant h (no per-step select in the hot loop).
  // Stage times are not needed: the models are autonomous (time argument ignored).
  ENS_REQUIRE_AUTONOMOUS(M, "fixed-step Tsit5 (stages evaluated at t = 0)");
  for (int64_t s = 0; s + 1 < steps; ++s) {
    tsit5_stages<M, V>(par, splat<V>(T(0)), hdt, ha, u, K, y);
    if (SAVE && next == s + 1) {
      if (SAVE == 3 && bulk)
        tsit5_save_bulk<n, V, T>(a, live, js, nb, next, s, y, blk0, reinterpret_cast<T*>(ens_fixed_smem));
      else
        tsit5_save_coded<n, V, T, SAVE == 1>(a, idx, live, js, next, s, a.dt0, u, K, y);
    }
#pragma unroll
    for (int j = 0; j < n; ++j) { u[j] = y[j]; K[0][j] = K[6][j]; }
  }
  {   // last step: h_last, lands on tf exactly
    const HaParam<V, C> hal{cf.hl};
    tsit5_stages<M, V>(par, splat<V>(T(0)), splat<V>(a.h_last), hal, u, K, y);
    if (SAVE && next == steps) {
      if (SAVE == 3 && bulk)
        tsit5_save_bulk<n, V, T>(a, live, js, nb, next, steps - 1, y, blk0, reinterpret_cast<T*>(ens_fixed_smem));
      else
        tsit5_save_coded<n, V, T, SAVE == 1>(a, idx, live, js, next, steps - 1, a.h_last, u, K, y);
    }
  }
  if constexpr (STATS) {   // statistics of the stored final states (u0 for lanes that diverged at t0)
    FinalPack<n, W, T> fp;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      fp.idx[w] = idx[w];
      fp.live[w] = live[w];
#pragma unroll
      for (int c = 0; c < n; ++c) fp.y[c][w] = lane(y[c], w);
    }
    fused_final_stats<n, W, T>(a.N, a.ld, a.u0, a.partial, i0, fp);
    if (!any) return;
  }
  if (SAVE == 3 && bulk && threadIdx.x == 0) bulk_wait_all();
  if (SAVE) {
    V nanv[n];
#pragma unroll
    for (int j = 0; j < n; ++j) nanv[j] = splat<V>(nanT<T>());
    for (; js < a.k; ++js) store_lanes<n, V, T>(a, idx, live, js, nanv);
  } else {
    store_lanes<n, V, T>(a, idx, live, 0, y);
  }
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (live[w]) {
      if (a.retcode) a.retcode[idx[w]] = lane_finite<n, V>(y, w) ? RET_SUCCESS : RET_DIVERGED;
      if (a.nacc) a.nacc[idx[w]] = (int32_t)steps;
      if (a.nrej) a.nrej[idx[w]] = 0;
    }
}

// ----------------------------------------------------------------- adaptive --
// Integrator state of one lane; init / step / finish are used both by the
// static one-trajectory-per-thread kernel and by the warp-refill scheduler.
template <class M, class T, bool SAVE> struct Tsit5Lane {
  static constexpr int n = M::n;
  T u[n], par[M::m], K[7][n];
  T t, h, lq_old;   // lq_old = log2 q_old (DESIGN R2)
  int32_t nacc, nrej, ret;
  int32_t js;
  bool done;

  __device__ __forceinline__ void init(const Args<T>& a, int64_t i) {
    load_column<M, T>(a, i, u, par);
    t = a.t0;
    h = a.dt0;                 // (T)min(dt, tf − t0), computed on the host in fp64
    lq_old = T(kLFloor);
    nacc = nrej = 0; ret = RET_SUCCESS; js = 0; done = false;
    M::f(u, par, t, K[0]);
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
    }
    if (!all_finite<n>(K[0])) { ret = RET_DIVERGED; done = true; }
    else if (!(t < a.tf)) done = true;
  }

  // One attempted step: stages, error, q, accept/reject, PI.
  __device__ __forceinline__ void step(const Args<T>& a, int64_t i) {
    if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
    const bool last = (t + h >= a.tf);
    if (last) h = a.tf - t;
    T y[n], E[n];
    const HaReg<T> ha(h);
    tsit5_stages<M, T>(par, t, h, ha, u, K, y);
    tsit5_error<n, T>(h, K, E);
    const T q2 = error_q2<n, T>(E, u, y, a.abstol, a.reltol);
    if (q2 < T(1)) {
      T tn = last ? a.tf : t + h;
      bool event = false;
      if constexpr (HasEvent<M>::value) {
        // DESIGN R18: sample the condition at θ_j = j/10 of the accepted step's
        // interpolant; in the first downward-crossing bracket, a fixed number of
        // bisections; the step ends at the crossing, where the affect applies.
        T gprev = M::event_g(u), thprev = T(0);
        for (int j = 1; j <= kEventPts && !event; ++j) {
          const T th = (j == kEventPts) ? T(1) : (T)j / (T)kEventPts;
          T xj[n];
          if (j == kEventPts) {
#pragma unroll
            for (int c = 0; c < n; ++c) xj[c] = y[c];
          } else {
            tsit5_interp<n, T>(th, h, u, K, xj);
          }
          const T gj = M::event_g(xj);
          if (gprev > T(0) && gj <= T(0)) {
            T lo = thprev, hi = th;
            for (int it = 0; it < (sizeof(T) == 4 ? 24 : 52); ++it) {
              const T mid = (lo + hi) * T(0.5);
              T xm[n];
              tsit5_interp<n, T>(mid, h, u, K, xm);
              if (M::event_g(xm) > T(0)) lo = mid; else hi = mid;
            }
            if (hi != T(1)) {
              tsit5_interp<n, T>(hi, h, u, K, y);     // y ← state at the crossing
              tn = t + hi * h;
            }
            event = true;
          }
          gprev = gj; thprev = th;
        }
      }
      if (SAVE) {
        const int64_t id[1] = {i};
        const bool lv[1] = {true};
        tsit5_save<n, T, T>(a, id, lv, js, t, tn, h, u, K, y);
      }
      t = tn;
      if constexpr (HasEvent<M>::value) {
        if (event) {
          M::affect(y, par);
#pragma unroll
          for (int j = 0; j < n; ++j) u[j] = y[j];
          M::f(u, par, t, K[0]);                       // FSAL no longer valid after the affect
        } else {
#pragma unroll
          for (int j = 0; j < n; ++j) { u[j] = y[j]; K[0][j] = K[6][j]; }
        }
      } else {
#pragma unroll
        for (int j = 0; j < n; ++j) { u[j] = y[j]; K[0][j] = K[6][j]; }
      }
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, 7.0 / 50.0, 2.0 / 25.0);
    } else {
      h = pi_reject<T>(h, q2, 7.0 / 50.0);
      ++nrej;
    }
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  __device__ __forceinline__ void finish(const Args<T>& a, int64_t i) {
    if (SAVE) {
      T nanv[n];
#pragma unroll
      for (int j = 0; j < n; ++j) nanv[j] = nanT<T>();
      for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
    } else {
      store_point<n>(a, i, 0, u);
    }
    if (a.retcode) a.retcode[i] = ret;
    if (a.nacc) a.nacc[i] = nacc;
    if (a.nrej) a.nrej[i] = nrej;
  }
};

// Static adaptive Tsit5 (one trajectory per thread, models without events), the
// loop written out with local state: per attempt exactly Tsit5Lane::step's
// operations, without the lane struct's done flag and early return.
template <class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) tsit5_static_kernel(const Args<T> a) {
  constexpr int n = M::n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  T u[n], par[M::m], K[7][n];
  load_column<M, T>(a, i, u, par);
  T t = a.t0, h = a.dt0, lq_old = T(kLFloor);
  int32_t nacc = 0, nrej = 0, ret = RET_SUCCESS;
  int js = 0;
  M::f(u, par, t, K[0]);
  if (SAVE) {
    while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
  }
  if (!all_finite<n>(K[0])) ret = RET_DIVERGED;
  else {
    const int64_t id[1] = {i};
    const bool lv[1] = {true};
    while (t < a.tf) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; break; }
      const bool last = (t + h >= a.tf);
      if (last) h = a.tf - t;
      T y[n], E[n];
      const HaReg<T> ha(h);
      tsit5_stages<M, T>(par, t, h, ha, u, K, y);
      tsit5_error<n, T>(h, K, E);
      const T q2 = error_q2<n, T>(E, u, y, a.abstol, a.reltol);
      if (q2 < T(1)) {
        const T tn = last ? a.tf : t + h;
        if (SAVE) tsit5_save<n, T, T>(a, id, lv, js, t, tn, h, u, K, y);
        t = tn;
#pragma unroll
        for (int j = 0; j < n; ++j) { u[j] = y[j]; K[0][j] = K[6][j]; }
        ++nacc;
        h = pi_accept<T>(h, q2, lq_old, 7.0 / 50.0, 2.0 / 25.0);
      } else {
        h = pi_reject<T>(h, q2, 7.0 / 50.0);
        ++nrej;
      }
      if (t < a.tf && t + h == t) { ret = RET_DTMIN; break; }
    }
  }
  if (SAVE) {
    T nanv[n];
#pragma unroll
    for (int j = 0; j < n; ++j) nanv[j] = nanT<T>();
    for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
  } else {
    store_point<n>(a, i, 0, u);
  }
  if (a.retcode) a.retcode[i] = ret;
  if (a.nacc) a.nacc[i] = nacc;
  if (a.nrej) a.nrej[i] = nrej;
}

// ------------------------------------------- adaptive fp32, component pairs --
// Static adaptive Tsit5 in fp32 with the stage, coefficient and error sums of
// components (0,1), (2,3), … as packed FFMA2 / FMUL2 lanes: the per-step
// products h·a_il are formed two at a time (FMUL2 of the broadcast h with a
// coefficient pair), and every stage FMA of a component pair is one FFMA2 whose
// coefficient operand is the scalar product broadcast to both lanes (SASS
// `R.F32` operand, no pack). Each lane rounds exactly like the scalar
// __fmul_rn / __fmaf_rn of tsit5_static_kernel in the same order, so the results
// are bit-identical; the RHS, the error norm, the controller and the saves read
// the pair halves as scalars. Cuts the issue count of an attempted Lorenz step
// from 283 to ≈240 (the kernel is issue-bound).
template <int n> struct PairV {
  static constexpr int P = n / 2, R = n % 2;
  float2 p[P > 0 ? P : 1];
  float s;   // component n − 1 when n is odd
  __device__ __forceinline__ float get(int c) const {
    if (R && c == n - 1) return s;
    return (c & 1) ? p[c >> 1].y : p[c >> 1].x;
  }
  __device__ __forceinline__ void to(float (&o)[n]) const {
#pragma unroll
    for (int c = 0; c < n; ++c) o[c] = get(c);
  }
  __device__ __forceinline__ void from(const float (&o)[n]) {
#pragma unroll
    for (int q = 0; q < P; ++q) p[q] = make_float2(o[2 * q], o[2 * q + 1]);
    if (R) s = o[n - 1];
  }
};
__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }
struct TsA2 { float2 v[11]; };
__host__ __device__ constexpr TsA2 make_ts_a2() {   // (a_il) in ts_idx order, rounded to float, paired
  TsA2 t{};
  float f[22] = {};
  for (int i = 1; i < 7; ++i)
    for (int l = 0; l < i; ++l) f[ts_idx(i, l)] = (float)ts_a(i, l);
  for (int x = 0; x < 11; ++x) t.v[x] = float2{f[2 * x], f[2 * x + 1]};
  return t;
}
static __constant__ TsA2 c_ts_a2 = make_ts_a2();

template <class M, bool SAVE>
__global__ void __launch_bounds__(256) tsit5_static_pair_kernel(const Args<float> a) {
  constexpr int n = M::n;
  using PV = PairV<n>;
  constexpr int P = PV::P;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  float us[n], par[M::m];
  load_column<M, float>(a, i, us, par);
  PV u, K[7];
  u.from(us);
  float t = a.t0, h = a.dt0, lq_old = float(kLFloor);
  int32_t nacc = 0, nrej = 0, ret = RET_SUCCESS;
  int js = 0;
  {
    float k0[n];
    M::f(us, par, t, k0);
    K[0].from(k0);
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, us); ++js; }
    }
    if (!all_finite<n>(k0)) ret = RET_DIVERGED;
  }
  if (ret == RET_SUCCESS) {
    const int64_t id[1] = {i};
    const bool lv[1] = {true};
    ENS_REQUIRE_AUTONOMOUS(M, "packed adaptive Tsit5 (stages evaluated at t = 0)");
    while (t < a.tf) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; break; }
      const bool last = (t + h >= a.tf);
      if (last) h = a.tf - t;
      // h·a_il, 21 products formed as 11 FMUL2 of the broadcast h with a coefficient
      // pair from the constant bank (the last lane of the last pair unused)
      float ha[22];
#pragma unroll
      for (int x = 0; x < 11; ++x) {
        const float2 r = __fmul2_rn(bc2(h), c_ts_a2.v[x]);
        ha[2 * x] = r.x;
        ha[2 * x + 1] = r.y;
      }
      PV y;
#pragma unroll
      for (int st = 1; st < 7; ++st) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
          float2 acc = u.p[q];
#pragma unroll
          for (int l = 0; l < st; ++l) acc = __ffma2_rn(bc2(ha[ts_idx(st, l)]), K[l].p[q], acc);
          y.p[q] = acc;
        }
        if (PV::R) {
          float acc = u.s;
#pragma unroll
          for (int l = 0; l < st; ++l) acc = __fmaf_rn(ha[ts_idx(st, l)], K[l].s, acc);
          y.s = acc;
        }
        float ys[n], o[n];
        y.to(ys);
        M::f(ys, par, 0.0f, o);
        K[st].from(o);
      }
      // E = h Σ b̃_l k_l (tsit5_error's order per component)
      float E[n];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        float2 e = __fmul2_rn(bc2((float)ts_bt(0)), K[0].p[q]);
#pragma unroll
        for (int l = 1; l < 7; ++l) e = __ffma2_rn(bc2((float)ts_bt(l)), K[l].p[q], e);
        e = __fmul2_rn(bc2(h), e);
        E[2 * q] = e.x;
        E[2 * q + 1] = e.y;
      }
      if (PV::R) {
        float e = (float)ts_bt(0) * K[0].s;
#pragma unroll
        for (int l = 1; l < 7; ++l) e = __fmaf_rn((float)ts_bt(l), K[l].s, e);
        E[n - 1] = h * e;
      }
      float ucur[n], ynew[n];
      u.to(ucur);
      y.to(ynew);
      const float q2 = error_q2<n, float>(E, ucur, ynew, a.abstol, a.reltol);
      if (q2 < 1.0f) {
        const float tn = last ? a.tf : t + h;
        if (SAVE) {
          float Ks[7][n];
#pragma unroll
          for (int l = 0; l < 7; ++l) K[l].to(Ks[l]);
          tsit5_save<n, float, float>(a, id, lv, js, t, tn, h, ucur, Ks, ynew);
        }
        t = tn;
        u = y;
        K[0] = K[6];
        ++nacc;
        h = pi_accept<float>(h, q2, lq_old, 7.0 / 50.0, 2.0 / 25.0);
      } else {
        h = pi_reject<float>(h, q2, 7.0 / 50.0);
        ++nrej;
      }
      if (t < a.tf && t + h == t) { ret = RET_DTMIN; break; }
    }
  }
  u.to(us);
  if (SAVE) {
    float nanv[n];
#pragma unroll
    for (int j = 0; j < n; ++j) nanv[j] = nanT<float>();
    for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
  } else {
    store_point<n>(a, i, 0, us);
  }
  if (a.retcode) a.retcode[i] = ret;
  if (a.nacc) a.nacc[i] = nacc;
  if (a.nrej) a.nrej[i] = nrej;
}

// Host-side construction of the fixed-step coefficient table (products in T).
template <class T, class C>
inline TsitCoef<C> make_tsit_coef(T h, T hl) {
  TsitCoef<C> cf;
  for (int i = 1; i < 7; ++i)
    for (int l = 0; l < i; ++l) {
      const T a = (T)ts_a(i, l);
      const T x = h * a, y = hl * a;
      if constexpr (sizeof(C) == 2 * sizeof(T)) {
        cf.h[ts_idx(i, l)] = C{x, x};
        cf.hl[ts_idx(i, l)] = C{y, y};
      } else {
        cf.h[ts_idx(i, l)] = x;
        cf.hl[ts_idx(i, l)] = y;
      }
    }
  return cf;
}

}  // namespace ens
