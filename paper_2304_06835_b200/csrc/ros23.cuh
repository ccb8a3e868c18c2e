// ros23.cuh — per-thread Rosenbrock23 (ode23s) stiff integrator for sm_100a.
//
// P:124-138 general Rosenbrock form; the method named in P:321 is the
// Shampine–Reichelt ode23s pair (DESIGN R10): one exact Jacobian (analytic
// functor instead of the paper's in-kernel forward AD), one LU of
// W = I − h d J with partial pivoting and three triangular solves per step —
// no Newton iteration, so no data-dependent branching.
// J, W, its LU and all stage vectors stay in registers (the paper's per-thread
// block of the block-diagonal W).
#pragma once
#include "common.cuh"
#include "models_stiff.cuh"

namespace ens {

__host__ __device__ constexpr double r23_d() { return 0.29289321881345248; }   // 1/(2+√2)
__host__ __device__ constexpr double r23_e32() { return 7.414213562373095; }   // 6+√2
__host__ __device__ constexpr double r23_inv12d() { return 1.0 / (1.0 - 2.0 * 0.29289321881345248); }

template <int n> constexpr bool kBranchSwap = (n > 4);

// In-register LU with partial pivoting; row swaps are predicated selects
// (no dynamically indexed arrays → no local memory). Canonical order DESIGN §4.
template <int n, class T>
__device__ __forceinline__ bool lu_factor(T (&A)[n][n], int (&piv)[n], T (&inv)[n]) {
  bool ok = true;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int kk = 0; kk < n; ++kk) {
    int pr = kk;
    T best = absT(A[kk][kk]);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int i = kk + 1; i < n; ++i) {
      const T v = absT(A[i][kk]);
      if (v > best) { best = v; pr = i; }
    }
    piv[kk] = pr;
    // For n > 4 the swap is a branch around the selects: the lanes of a warp
    // mostly agree on the pivot row (neighbouring trajectories, similar W), so a
    // warp with no swap at this column skips the row exchange entirely (HIRES /
    // POLLU 12–26 % faster). For n ≤ 4 plain selects measured faster (OREGO,
    // refill Rosenbrock23 on C3: 5–10 %).
    if (!kBranchSwap<n> || pr != kk) {
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int i = kk + 1; i < n; ++i) {
        const bool sw = (pr == i);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
        for (int j = 0; j < n; ++j) {
          const T a0 = A[kk][j], a1 = A[i][j];
          A[kk][j] = sw ? a1 : a0;
          A[i][j] = sw ? a0 : a1;
        }
      }
    }
    const T pivot = A[kk][kk];
    ok = ok && (pivot != T(0)) && finiteT(pivot);
    inv[kk] = T(1) / pivot;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int i = kk + 1; i < n; ++i) {
      const T l = A[i][kk] * inv[kk];
      A[i][kk] = l;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = kk + 1; j < n; ++j) A[i][j] = fmaT(-l, A[kk][j], A[i][j]);
    }
  }
  return ok;
}

// PERM = false: the factorization took no row exchange (identity permutation).
template <int n, class T, bool PERM = true>
__device__ __forceinline__ void lu_solve(const T (&LU)[n][n], const int (&piv)[n], const T (&inv)[n], const T (&b)[n],
                                         T (&x)[n]) {
  T z[n];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int i = 0; i < n; ++i) z[i] = b[i];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int kk = 0; kk < n; ++kk) {
    if (PERM && (!kBranchSwap<n> || piv[kk] != kk)) {   // branch for n > 4, as in lu_factor
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int i = kk + 1; i < n; ++i) {
        const bool sw = (piv[kk] == i);
        const T z0 = z[kk], z1 = z[i];
        z[kk] = sw ? z1 : z0;
        z[i] = sw ? z0 : z1;
      }
    }
  }
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int i = 0; i < n; ++i) {          // forward, unit lower
    T s = z[i];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int j = 0; j < i; ++j) s = fmaT(-LU[i][j], z[j], s);
    z[i] = s;
  }
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int i = n - 1; i >= 0; --i) {     // backward
    T s = z[i];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int j = i + 1; j < n; ++j) s = fmaT(-LU[i][j], x[j], s);
    x[i] = s * inv[i];
  }
}

// LU of W = build() with partial pivoting, warp-uniform fast path for n ≤ 4:
// the factorization first runs WITHOUT row exchanges while checking the
// pivoting rule (row i would be exchanged at column k iff |A_ik| > |A_kk| for
// some i > k, the first-maximum rule of lu_factor); if no lane of the warp
// needed an exchange, the result is exactly lu_factor's (same operations, same
// order) and the solves skip the permutation (Robertson's W = I − h d J never
// needs one: a diagonal entry dominates each column); otherwise W is rebuilt
// and factored with exchanges. `permuted` is warp-uniform, so the solves'
// branch on it does not diverge. Models whose W needs exchanges often declare
// `lu_fast_path = false` (OREGO: its second column in ≈9 % of the sampled
// steps; the rebuild then costs more than the exchanges save) and, like n > 4,
// take lu_factor directly. (Continuing with exchanges from the first column
// that needs one, instead of rebuilding, measured slower on C3 and OREGO.)
template <class M, class = void> struct LuFastPath { static constexpr bool value = true; };
template <class M> struct LuFastPath<M, decltype((void)M::lu_fast_path)> { static constexpr bool value = M::lu_fast_path; };

template <class M, int n, class T, class Build>
__device__ __forceinline__ bool lu_factor_fast(T (&A)[n][n], int (&piv)[n], T (&inv)[n], bool& permuted,
                                               Build&& build) {
  build(A);
  permuted = true;
  if constexpr (kBranchSwap<n> || !LuFastPath<M>::value) {
    return lu_factor<n, T>(A, piv, inv);
  } else {
    bool need = false, ok = true;
#pragma unroll
    for (int kk = 0; kk < n; ++kk) {
      const T d = absT(A[kk][kk]);
#pragma unroll
      for (int i = kk + 1; i < n; ++i) need = need || (absT(A[i][kk]) > d);
      piv[kk] = kk;
      const T pivot = A[kk][kk];
      ok = ok && (pivot != T(0)) && finiteT(pivot);
      inv[kk] = T(1) / pivot;
#pragma unroll
      for (int i = kk + 1; i < n; ++i) {
        const T l = A[i][kk] * inv[kk];
        A[i][kk] = l;
#pragma unroll
        for (int j = kk + 1; j < n; ++j) A[i][j] = fmaT(-l, A[kk][j], A[i][j]);
      }
    }
    permuted = __any_sync(__activemask(), need);
    if (permuted) {
      build(A);
      ok = lu_factor<n, T>(A, piv, inv);
    }
    return ok;
  }
}

template <int n, class T>
__device__ __forceinline__ void lu_solve_w(const T (&LU)[n][n], const int (&piv)[n], const T (&inv)[n], bool permuted,
                                           const T (&b)[n], T (&x)[n]) {
  if constexpr (kBranchSwap<n>) {
    lu_solve<n, T, true>(LU, piv, inv, b, x);   // n > 4: always lu_factor (no fast path)
  } else {
    if (permuted) lu_solve<n, T, true>(LU, piv, inv, b, x);
    else lu_solve<n, T, false>(LU, piv, inv, b, x);
  }
}

// One ode23s step. F0 = f(u,t) (FSAL). Outputs u_new, F2 = f(u_new), k1, k2, E.
template <class M, class T>
__device__ __forceinline__ bool ros23_step(const T (&par)[M::m], T t, T h, const T (&u)[M::n], const T (&F0)[M::n],
                                           T (&un)[M::n], T (&F2)[M::n], T (&k1)[M::n], T (&k2)[M::n],
                                           T (&E)[M::n]) {
  ENS_REQUIRE_AUTONOMOUS(M, "Rosenbrock23 (no h·d·∂f/∂t term, P:125-136)");
  constexpr int n = M::n;
  const T d = T(r23_d()), e32 = T(r23_e32());
  T W[n][n];
  const T hd = h * d;
  int piv[n];
  T inv[n];
  bool pm;
  const bool ok = lu_factor_fast<M, n, T>(W, piv, inv, pm, [&](T (&A)[n][n]) {
    model_jacobian<M, T>(u, par, t, A);       // J (hand-written or forward-mode AD)
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int i = 0; i < n; ++i)
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) A[i][j] = (i == j ? T(1) : T(0)) - hd * A[i][j];   // W = I − h d J
  });
  lu_solve_w<n, T>(W, piv, inv, pm, F0, k1);  // k1 = W⁻¹ F0
  T y[n], F1[n], r[n], k3[n];
  const T hh = h * T(0.5);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) y[j] = fmaT(hh, k1[j], u[j]);
  M::f(y, par, t + hh, F1);                  // F1 = f(u + h/2 k1)
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) r[j] = F1[j] - k1[j];
  lu_solve_w<n, T>(W, piv, inv, pm, r, k2);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) k2[j] = k2[j] + k1[j];   // k2 = W⁻¹(F1 − k1) + k1
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) un[j] = fmaT(h, k2[j], u[j]);
  M::f(un, par, t + h, F2);                  // F2 = f(u_new)
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) {
    const T aa = fmaT(-e32, k2[j] - F1[j], F2[j]);
    r[j] = fmaT(T(-2), k1[j] - F0[j], aa);   // F2 − e32(k2 − F1) − 2(k1 − F0)
  }
  lu_solve_w<n, T>(W, piv, inv, pm, r, k3);
  const T h6 = h * T(1.0 / 6.0);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) E[j] = h6 * (fmaT(T(-2), k2[j], k1[j]) + k3[j]);   // E = h/6 (k1 − 2k2 + k3)
  return ok;
}

template <int n, class T>
__device__ __forceinline__ void ros23_interp(T theta, T h, const T (&u)[n], const T (&k1)[n], const T (&k2)[n],
                                             T (&o)[n]) {
  const T d = T(r23_d()), inv12d = T(r23_inv12d());
  const T c1 = (theta * (T(1) - theta)) * inv12d;
  const T c2 = (theta * (theta - T(2) * d)) * inv12d;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int j = 0; j < n; ++j) o[j] = fmaT(h, fmaT(c2, k2[j], c1 * k1[j]), u[j]);
}

template <int n, class T>
__device__ __forceinline__ void ros23_save(const Args<T>& a, int64_t i, int& js, T t, T tn, T h, const T (&u)[n],
                                           const T (&k1)[n], const T (&k2)[n], const T (&un)[n]) {
  while (js < a.k) {
    const T tau = __ldg(a.tau + js);
    if (!(tau <= tn)) break;
    if (tau == tn) {
      store_point<n>(a, i, js, un);
    } else {
      T o[n];
      ros23_interp<n, T>((tau - t) / h, h, u, k1, k2, o);
      store_point<n>(a, i, js, o);
    }
    ++js;
  }
}

template <class M, class T, bool SAVE> struct Ros23Lane {
  static constexpr int n = M::n;
  T u[n], par[M::m], F0[n];
  T t, h, lq_old;   // lq_old = log2 q_old (DESIGN R2)
  int32_t nacc, nrej, ret, js;
  bool done;

  __device__ __forceinline__ void init(const Args<T>& a, int64_t i) {
    load_column<M, T>(a, i, u, par);
    t = a.t0; h = a.dt0; lq_old = T(kLFloor);
    nacc = nrej = 0; ret = RET_SUCCESS; js = 0; done = false;
    M::f(u, par, t, F0);
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
    }
    if (!all_finite<n>(F0)) { ret = RET_DIVERGED; done = true; }
    else if (!(t < a.tf)) done = true;
  }

  __device__ __forceinline__ void step(const Args<T>& a, int64_t i) {
    if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
    const bool last = (t + h >= a.tf);
    if (last) h = a.tf - t;
    T un[n], F2[n], k1[n], k2[n], E[n];
    if (!ros23_step<M, T>(par, t, h, u, F0, un, F2, k1, k2, E)) {
      h = h * T(0.5);                       // singular W: reject and halve (DESIGN R10)
      ++nrej;
      if (t + h == t) { ret = RET_SINGULAR; done = true; }
      return;
    }
    const T q2 = error_q2<n, T>(E, u, un, a.abstol, a.reltol);
    if (q2 < T(1)) {
      const T tn = last ? a.tf : t + h;
      if (SAVE) ros23_save<n, T>(a, i, js, t, tn, h, u, k1, k2, un);
      t = tn;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) { u[j] = un[j]; F0[j] = F2[j]; }
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, 7.0 / 20.0, 2.0 / 10.0);
    } else {
      h = pi_reject<T>(h, q2, 7.0 / 20.0);
      ++nrej;
    }
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  __device__ __forceinline__ void finish(const Args<T>& a, int64_t i) {
    if (SAVE) {
      T nanv[n];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
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

// Static adaptive Rosenbrock23 (one trajectory per thread), the loop written out with
// local state: the same per-attempt operations as Ros23Lane (which the refill
// scheduler keeps), without the lane struct's done flag and early return, whose
// merge points cost ≈30 register moves per attempt (profiles: C3 12.28 → 11.9 ms).
template <class M, class T, bool SAVE, int MINB>
__global__ void __launch_bounds__(256, MINB) ros23_static_kernel(const Args<T> a) {
  constexpr int n = M::n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  T u[n], par[M::m], F0[n];
  load_column<M, T>(a, i, u, par);
  T t = a.t0, h = a.dt0, lq_old = T(kLFloor);
  int32_t nacc = 0, nrej = 0, ret = RET_SUCCESS;
  int js = 0;
  M::f(u, par, t, F0);
  if (SAVE) {
    while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
  }
  if (!all_finite<n>(F0)) ret = RET_DIVERGED;
  else {
    while (t < a.tf) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; break; }
      const bool last = (t + h >= a.tf);
      if (last) h = a.tf - t;
      T un[n], F2[n], k1[n], k2[n], E[n];
      if (!ros23_step<M, T>(par, t, h, u, F0, un, F2, k1, k2, E)) {
        h = h * T(0.5);
        ++nrej;
        if (t + h == t) { ret = RET_SINGULAR; break; }
        continue;
      }
      const T q2 = error_q2<n, T>(E, u, un, a.abstol, a.reltol);
      if (q2 < T(1)) {
        const T tn = last ? a.tf : t + h;
        if (SAVE) ros23_save<n, T>(a, i, js, t, tn, h, u, k1, k2, un);
        t = tn;
#pragma unroll
        for (int j = 0; j < n; ++j) { u[j] = un[j]; F0[j] = F2[j]; }
        ++nacc;
        h = pi_accept<T>(h, q2, lq_old, 7.0 / 20.0, 2.0 / 10.0);
      } else {
        h = pi_reject<T>(h, q2, 7.0 / 20.0);
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

// Fixed-step Rosenbrock23 on the DESIGN R3 grid (used for the order /
// stability pins); a singular W ends the trajectory with RET_SINGULAR.
template <class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) ros23_fixed_kernel(const Args<T> a) {
  constexpr int n = M::n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  T u[n], par[M::m], F0[n];
  load_column<M, T>(a, i, u, par);
  M::f(u, par, a.t0, F0);
  int js = 0;
  if (SAVE) {
    while (js < a.k && __ldg(a.tau + js) <= a.t0) { store_point<n>(a, i, js, u); ++js; }
  }
  int32_t ret = RET_SUCCESS, nacc = 0;
  if (!all_finite<n>(F0)) ret = RET_DIVERGED;
  else {
    for (int64_t s = 0; s < a.nsteps; ++s) {
      const bool last = (s == a.nsteps - 1);
      const T h = last ? a.h_last : a.dt0;
      const T t = (T)(a.t0d + (double)s * a.dtd);
      T un[n], F2[n], k1[n], k2[n], E[n];
      if (!ros23_step<M, T>(par, t, h, u, F0, un, F2, k1, k2, E)) { ret = RET_SINGULAR; break; }
      if (SAVE) ros23_save<n, T>(a, i, js, t, last ? a.tf : (T)(a.t0d + (double)(s + 1) * a.dtd), h, u, k1, k2, un);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) { u[j] = un[j]; F0[j] = F2[j]; }
      ++nacc;
    }
    if (ret == RET_SUCCESS && !all_finite<n>(u)) ret = RET_DIVERGED;
  }
  if (SAVE) {
    T nanv[n];
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int j = 0; j < n; ++j) nanv[j] = nanT<T>();
    for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
  } else {
    store_point<n>(a, i, 0, u);
  }
  if (a.retcode) a.retcode[i] = ret;
  if (a.nacc) a.nacc[i] = nacc;
  if (a.nrej) a.nrej[i] = 0;
}

}  // namespace ens
