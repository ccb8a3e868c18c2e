// group.cuh — G lanes per trajectory for the Rodas methods on the larger stiff
// systems (HIRES n = 8, POLLU n = 20, NEXT-4 / NEXT-2).
//
// One thread per trajectory (the paper's EnsembleGPUKernel) keeps W, its LU and
// every stage vector of one trajectory in one thread's registers. For n = 8 / 20
// that is 120–255 registers plus spill slots, and the stiff suite's 8192
// trajectories are then 1.7 warps per SM: the kernel is latency-bound with the
// SMs mostly idle. Here a group of G = 8 / 16 / 32 lanes (the
// next power of two ≥ n) carries one trajectory: lane r holds row r of W (then of
// its LU) and component r of every vector, so an 8192-trajectory ensemble fills
// the GPU with 32·8192 / G threads.
//
// The arithmetic is the per-thread kernel's, operation for operation,
// so results are bit-identical to it (and to the oracle):
//   * J: lane r forms column r by a one-seed forward-mode AD pass (ad.cuh: every
//     partial has its own chain of the dual rules, so a column does not depend on
//     which pass computes it); the columns are transposed to rows through shared
//     memory; W = I/(hγ) − J row by row.
//   * LU with partial pivoting (lu_factor): the pivot of column k is the first
//     position with the largest |A_ik| (a butterfly max over (value, position)
//     with the serial scan's NaN rule); rows do not move — each lane tracks the
//     logical position of its row, and a row exchange swaps two positions, which
//     is what the serial code's full-row swap amounts to. The pivot row is
//     broadcast and every lower row updates itself with the serial fma.
//   * Solves: forward substitution in rounds j = 0..n−1 (the final z_j broadcast,
//     every later row one fma — the serial ascending order per row); back
//     substitution in rounds i = n−1..0, the row at position i summing its
//     ascending terms over the broadcast x_j (j > i) exactly as the serial loop.
//   * RHS: the stage vector is gathered into every lane, f is evaluated in full
//     by every lane (same operations) and each lane keeps its component.
//   * Error norm: each lane forms its quotient; every lane sums the n squares in
//     component order (error_q2's fma chain), so q² and the controller are
//     replicated bit for bit across the group.
#pragma once
#include "rodas.cuh"

namespace ens {

template <int n> constexpr int kGroupWidth = n <= 8 ? 8 : n <= 16 ? 16 : 32;
// the models that take the group kernels: forward-mode-AD Jacobians with n > 4 (HIRES, POLLU)
template <class M> constexpr bool kUseGroup = HasAdJac<M>::value && (M::n > 4) && (M::n <= 32);

template <int G> struct Grp {
  unsigned mask;   // the group's lanes
  int r;           // lane within the group = row / component index
  __device__ __forceinline__ Grp() {
    const int lane = threadIdx.x & 31;
    r = lane & (G - 1);
    mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  }
  template <class V> __device__ __forceinline__ V bc(V v, int src) const { return __shfl_sync(mask, v, src, G); }
  template <class V> __device__ __forceinline__ V bx(V v, int off) const { return __shfl_xor_sync(mask, v, off, G); }
};

// all components of a distributed vector in every lane
template <int n, int G, class T>
__device__ __forceinline__ void grp_gather(const Grp<G>& g, T v, T (&full)[n]) {
#pragma unroll
  for (int j = 0; j < n; ++j) full[j] = g.bc(v, j);
}
// component r of a replicated vector (r < n; 0 for the idle lanes r ≥ n)
template <int n, class T>
__device__ __forceinline__ T grp_pick(const T (&full)[n], int r) {
  T v = T(0);
#pragma unroll
  for (int j = 0; j < n; ++j) v = (r == j) ? full[j] : v;
  return v;
}

// Row-layout LU of one trajectory's W (lane r: row r of W on entry).
template <int n, class T, int G> struct GrpLU {
  T R[n];          // this lane's row (W, then L \ U)
  int pos;         // its logical row position after the row exchanges so far
  int lane_of[n];  // lane holding logical position k (replicated)
  T inv_own;       // 1 / pivot of this lane's final position

  // lu_factor (ros23.cuh) on the group; false if a pivot is zero or non-finite
  __device__ __forceinline__ bool factor(const Grp<G>& g) {
    bool ok = true;
    pos = g.r;
    inv_own = T(0);
#pragma unroll
    for (int kk = 0; kk < n; ++kk) {
      // pivot: the first position ≥ kk with the largest |A_ik| (serial scan: strict '>' from
      // best = |A_kk,kk|, so NaN entries are never chosen and a NaN at kk keeps kk)
      const bool cand = (pos >= kk) && (pos < n);
      T v = cand ? absT(R[kk]) : T(-1);
      if (cand && !(v == v)) v = (pos == kk) ? infT<T>() : T(-1);
      int key = (pos << 5) | g.r;
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) {
        const T ov = g.bx(v, off);
        const int ok_ = g.bx(key, off);
        if (ov > v || (ov == v && ok_ < key)) { v = ov; key = ok_; }
      }
      const int pr = key >> 5, pl = key & 31;
      if (pos == pr) pos = kk;
      else if (pos == kk) pos = pr;
      lane_of[kk] = pl;
      const T pivot = g.bc(R[kk], pl);
      ok = ok && (pivot != T(0)) && finiteT(pivot);
      const T inv = T(1) / pivot;
      if (pos == kk) inv_own = inv;
      T prow[n];
#pragma unroll
      for (int j = kk + 1; j < n; ++j) prow[j] = g.bc(R[j], pl);
      if (pos > kk && pos < n) {
        const T l = R[kk] * inv;
        R[kk] = l;
#pragma unroll
        for (int j = kk + 1; j < n; ++j) R[j] = fmaT(-l, prow[j], R[j]);
      }
    }
    return ok;
  }

  // lu_solve: b distributed (lane r: b_r) → x distributed (lane r: x_r)
  __device__ __forceinline__ T solve(const Grp<G>& g, T b) const {
    T s = b;   // z at this lane's position: the row exchanges applied to b move b_r with row r
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const T zj = g.bc(s, lane_of[j]);
      if (pos > j && pos < n) s = fmaT(-R[j], zj, s);
    }
    T xall[n];
    T xm = T(0);
#pragma unroll
    for (int q = 0; q < n; ++q) {     // positions i = n − 1 … 0 (static indices throughout)
      const int i = n - 1 - q;
      if (pos == i) {
        T t = s;
#pragma unroll
        for (int j = 0; j < n; ++j)
          if (j > i) t = fmaT(-R[j], xall[j], t);
        xm = t * inv_own;
      }
      xall[i] = g.bc(xm, lane_of[i]);
    }
    return grp_pick<n, T>(xall, g.r);
  }
};

// error_q2 (common.cuh) on distributed E, u, u_new: replicated q²
template <int n, int G, class T>
__device__ __forceinline__ T grp_error_q2(const Grp<G>& g, T E, T u, T un, T abstol, T reltol) {
  T rr = T(0);
  if (g.r < n) {
    const T sc = abstol + reltol * maxT_nn(absT(u), absT(un));
    rr = E / sc;
  }
  T s = T(0);
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const T rj = g.bc(rr, j);
    s = (j == 0) ? rj * rj : fmaT(rj, rj, s);
  }
  T q2 = s * T(1.0 / n);
  if (!finiteT(q2)) q2 = infT<T>();
  return q2;
}

// f at a distributed state: every lane evaluates f in full, keeps its component
template <class M, int G, class T>
__device__ __forceinline__ T grp_rhs(const Grp<G>& g, const T (&par)[M::m], T t, T y) {
  T yf[M::n], o[M::n];
  grp_gather<M::n, G, T>(g, y, yf);
  M::f(yf, par, t, o);
  return grp_pick<M::n, T>(o, g.r);
}

// rodas_step on the group. uf = u in every lane (for J), u / F0 distributed;
// outputs u_new and K[s] distributed. jbuf: this group's n×n shared-memory tile.
template <class Tab, class M, class T, int G>
__device__ __forceinline__ bool grp_rodas_step(const Grp<G>& g, const T (&par)[M::m], T t, T h, const T (&uf)[M::n],
                                               T u, T F0, T& un, T (&K)[Tab::S], T* jbuf) {
  ENS_REQUIRE_AUTONOMOUS(M, "Rodas (no γ_i·h·∂f/∂t terms, P:125-136)");
  constexpr int n = M::n, S = Tab::S;
  const T hg = h * T(Tab::gamma);
  const T ihg = T(1) / hg;
  const T ih = T(1) / h;
  // J column r by a one-seed AD pass, transposed to rows through shared memory
  if (g.r < n) {
    Dual<T, 1> y[n], o[n];
#pragma unroll
    for (int i = 0; i < n; ++i) { y[i].v = uf[i]; y[i].d[0] = (i == g.r) ? T(1) : T(0); }
    M::f(y, par, t, o);
#pragma unroll
    for (int i = 0; i < n; ++i) jbuf[i * n + g.r] = o[i].d[0];
  }
  __syncwarp(g.mask);
  GrpLU<n, T, G> lu;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const T Jrj = (g.r < n) ? jbuf[g.r * n + j] : T(0);
    lu.R[j] = (g.r == j ? ihg : T(0)) - Jrj;            // W = I/(hγ) − J
  }
  __syncwarp(g.mask);   // jbuf is rewritten by the next step
  const bool ok = lu.factor(g);
  K[0] = lu.solve(g, F0);                                 // k1 = W⁻¹ f(u)
  T y = u;
#pragma unroll
  for (int s = 1; s < S; ++s) {
    T hc[S - 1];
#pragma unroll
    for (int j = 0; j < s; ++j) hc[j] = T(Tab::c(s, j)) * ih;
    T acc = u;
#pragma unroll
    for (int j = 0; j < s; ++j) acc = fmaT(T(Tab::a(s, j)), K[j], acc);   // Y_s = u + Σ a_sj k_j
    y = acc;
    T rr = grp_rhs<M, G, T>(g, par, t, y);
#pragma unroll
    for (int j = 0; j < s; ++j) rr = fmaT(hc[j], K[j], rr);              // f(Y_s) + Σ (c_sj/h) k_j
    K[s] = lu.solve(g, rr);
  }
  un = y + K[S - 1];                                      // u_new = Y_S + k_S
  return ok;
}

// Adaptive Rodas4 / Rodas5 / Rodas5P, one trajectory per group (static mapping).
// DENSE = 0: Rodas4's continuous extension for saves (rodas4_interp);
// DENSE = 1: the R24 shortened step (rodas_saves).
template <class Tab, class M, class T, int G, bool SAVE, int DENSE>
__global__ void __launch_bounds__(256) rodas_group_kernel(const Args<T> a) {
  constexpr int n = M::n, S = Tab::S, NG = 256 / G;
  static_assert(n <= G && (DENSE == 1 || S == 6), "group width / dense-output mode");
  __shared__ T jtile[NG][n * n];
  const Grp<G> g;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if (i >= a.N) return;   // whole groups
  T* jbuf = jtile[threadIdx.x / G];
  const bool act = g.r < n;
  T par[M::m];
#pragma unroll
  for (int c = 0; c < M::m; ++c) par[c] = a.p_broadcast ? __ldg(a.p + c) : __ldg(a.p + (size_t)c * a.ld + i);
  T u = act ? __ldg(a.u0 + (size_t)g.r * a.ld + i) : T(0);
  T uf[n];
  grp_gather<n, G, T>(g, u, uf);
  T t = a.t0, h = a.dt0, lq_old = T(kLFloor);
  int32_t nacc = 0, nrej = 0, ret = RET_SUCCESS;
  int js = 0;
  T F0;
  {
    T o[n];
    M::f(uf, par, t, o);
    F0 = grp_pick<n, T>(o, g.r);
    if (!all_finite<n>(o)) ret = RET_DIVERGED;
  }
  if (SAVE) {
    while (js < a.k && __ldg(a.tau + js) <= t) {
      if (act) a.u_out[((size_t)js * n + g.r) * a.ldo + i] = u;
      ++js;
    }
  }
  if (ret == RET_SUCCESS) {
    while (t < a.tf) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; break; }
      const bool last = (t + h >= a.tf);
      if (last) h = a.tf - t;
      T un, K[S];
      if (!grp_rodas_step<Tab, M, T, G>(g, par, t, h, uf, u, F0, un, K, jbuf)) {
        h = h * T(0.5);                       // singular W: reject and halve (DESIGN R10)
        ++nrej;
        if (t + h == t) { ret = RET_SINGULAR; break; }
        continue;
      }
      const T q2 = grp_error_q2<n, G, T>(g, K[S - 1], u, un, a.abstol, a.reltol);
      if (q2 < T(1)) {
        const T tn = last ? a.tf : t + h;
        if (SAVE) {
          while (js < a.k) {
            const T tau = __ldg(a.tau + js);
            if (!(tau <= tn)) break;
            T o = un;
            if (!(tau == tn)) {
              if constexpr (DENSE == 0) {           // rodas4_interp, component r
                const T theta = (tau - t) / h, th1 = T(1) - theta;
                T s1 = T(rd_d(0, 0)) * K[0], s2 = T(rd_d(1, 0)) * K[0];
#pragma unroll
                for (int j = 1; j < 5; ++j) {
                  s1 = fmaT(T(rd_d(0, j)), K[j], s1);
                  s2 = fmaT(T(rd_d(1, j)), K[j], s2);
                }
                const T w = fmaT(th1, fmaT(theta, s2, s1), un);
                o = fmaT(th1, u, theta * w);
              } else {                              // R24: one step of length τ − t from (t, u)
                T Ks[S];
                if (!grp_rodas_step<Tab, M, T, G>(g, par, t, tau - t, uf, u, F0, o, Ks, jbuf)) o = nanT<T>();
              }
            }
            if (act) a.u_out[((size_t)js * n + g.r) * a.ldo + i] = o;
            ++js;
          }
        }
        t = tn;
        u = un;
        grp_gather<n, G, T>(g, u, uf);
        {
          T o[n];
          M::f(uf, par, t, o);
          F0 = grp_pick<n, T>(o, g.r);
        }
        ++nacc;
        h = pi_accept<T>(h, q2, lq_old, Tab::beta1, Tab::beta2);
      } else {
        h = pi_reject<T>(h, q2, Tab::beta1);
        ++nrej;
      }
      if (t < a.tf && t + h == t) { ret = RET_DTMIN; break; }
    }
  }
  if (act) {
    if (SAVE) {
      for (; js < a.k; ++js) a.u_out[((size_t)js * n + g.r) * a.ldo + i] = nanT<T>();
    } else {
      a.u_out[(size_t)g.r * a.ldo + i] = u;
    }
  }
  if (g.r == 0) {
    if (a.retcode) a.retcode[i] = ret;
    if (a.nacc) a.nacc[i] = nacc;
    if (a.nrej) a.nrej[i] = nrej;
  }
}

}  // namespace ens
