// rodas4.cuh — per-thread Rodas4 stiff integrator for sm_100a (GPURodas4,
// P:322-323; NEXT-2; DESIGN R20).
//
// Hairer & Wanner's RODAS tableau in W-form: one exact Jacobian (analytic or
// in-kernel forward AD), one in-register LU of W = I/(hγ) − J, six
// triangular solves and six RHS evaluations per step; stiffly accurate, so the
// embedded order-3 solution is Y6 and the error estimate is k6. Like
// Rosenbrock23 there is no Newton iteration. All stage
// vectors, J, W and its LU stay in registers for n ≤ 8.
#pragma once
#include "common.cuh"
#include "models_stiff.cuh"
#include "ros23.cuh"   // lu_factor / lu_solve

namespace ens {

__host__ __device__ constexpr double rd_gamma() { return 0.25; }
__host__ __device__ constexpr double rd_a(int s, int j) {
  constexpr double A[6][5] = {
      {0, 0, 0, 0, 0},
      {1.544, 0, 0, 0, 0},
      {0.9466785280815826, 0.2557011698983284, 0, 0, 0},
      {3.314825187068521, 2.896124015972201, 0.9986419139977817, 0, 0},
      {1.221224509226641, 6.019134481288629, 12.53708332932087, -0.6878860361058950, 0},
      {1.221224509226641, 6.019134481288629, 12.53708332932087, -0.6878860361058950, 1.0}};
  return A[s][j];
}
__host__ __device__ constexpr double rd_c(int s, int j) {
  constexpr double C[6][5] = {
      {0, 0, 0, 0, 0},
      {-5.6688, 0, 0, 0, 0},
      {-2.430093356833875, -0.2063599157091915, 0, 0, 0},
      {-0.1073529058151375, -9.594562251023355, -20.47028614809616, 0, 0},
      {7.496443313967647, -10.24680431464352, -33.99990352819905, 11.70890893206160, 0},
      {8.083246795921522, -7.981132988064893, -31.52159432874371, 16.31930543123136, -6.058818238834054}};
  return C[s][j];
}
__host__ __device__ constexpr double rd_d(int r, int j) {   // r = 0: D2 (s1), r = 1: D3 (s2)
  constexpr double D[2][5] = {
      {10.12623508344586, -7.487995877610167, -34.80091861555747, -7.992771707568823, 1.025137723295662},
      {-0.6762803392801253, 6.087714651680015, 16.43084320892478, 24.76722511418386, -6.594389125716872}};
  return D[r][j];
}

// One Rodas4 step (autonomous models). F0 = f(u). Outputs u_new and K = k1..k6
// (E = k6). Returns false if W is singular (the outputs are then meaningless).
template <class M, class T>
__device__ __forceinline__ bool rodas4_step(const T (&par)[M::m], T t, T h, const T (&u)[M::n],
                                            const T (&F0)[M::n], T (&un)[M::n], T (&K)[6][M::n]) {
  constexpr int n = M::n;
  T W[n][n];
  model_jacobian<M, T>(u, par, t, W);
  const T hg = h * T(rd_gamma());
  const T ihg = T(1) / hg;
  const T ih = T(1) / h;
#pragma unroll (n <= 8 ? n : 1)
  for (int i = 0; i < n; ++i)
#pragma unroll (n <= 8 ? n : 1)
    for (int j = 0; j < n; ++j) W[i][j] = (i == j ? ihg : T(0)) - W[i][j];   // W = I/(hγ) − J
  int piv[n];
  T inv[n];
  const bool ok = lu_factor<n, T>(W, piv, inv);
  lu_solve<n, T>(W, piv, inv, F0, K[0]);                                     // k1 = W⁻¹ f(u)
  T y[n], F[n], r[n];
#pragma unroll
  for (int s = 1; s < 6; ++s) {
    T hc[5];
#pragma unroll
    for (int j = 0; j < s; ++j) hc[j] = T(rd_c(s, j)) * ih;                  // c_sj / h
#pragma unroll (n <= 8 ? n : 1)
    for (int c = 0; c < n; ++c) {
      T acc = u[c];
#pragma unroll
      for (int j = 0; j < s; ++j) acc = fmaT(T(rd_a(s, j)), K[j][c], acc);  // Y_s = u + Σ a_sj k_j
      y[c] = acc;
    }
    M::f(y, par, t, F);
#pragma unroll (n <= 8 ? n : 1)
    for (int c = 0; c < n; ++c) {
      T acc = F[c];
#pragma unroll
      for (int j = 0; j < s; ++j) acc = fmaT(hc[j], K[j][c], acc);          // f(Y_s) + Σ (c_sj/h) k_j
      r[c] = acc;
    }
    lu_solve<n, T>(W, piv, inv, r, K[s]);
  }
#pragma unroll (n <= 8 ? n : 1)
  for (int c = 0; c < n; ++c) un[c] = y[c] + K[5][c];                        // u_new = Y6 + k6
  return ok;
}

// RODAS continuous extension: (1−θ)u + θ(u_new + (1−θ)(s1 + θ s2)).
template <int n, class T>
__device__ __forceinline__ void rodas4_interp(T theta, const T (&u)[n], const T (&un)[n], const T (&K)[6][n],
                                              T (&o)[n]) {
  const T th1 = T(1) - theta;
#pragma unroll (n <= 8 ? n : 1)
  for (int c = 0; c < n; ++c) {
    T s1 = T(rd_d(0, 0)) * K[0][c], s2 = T(rd_d(1, 0)) * K[0][c];
#pragma unroll
    for (int j = 1; j < 5; ++j) {
      s1 = fmaT(T(rd_d(0, j)), K[j][c], s1);
      s2 = fmaT(T(rd_d(1, j)), K[j][c], s2);
    }
    const T w = fmaT(th1, fmaT(theta, s2, s1), un[c]);
    o[c] = fmaT(th1, u[c], theta * w);
  }
}

template <int n, class T>
__device__ __forceinline__ void rodas4_save(const Args<T>& a, int64_t i, int& js, T t, T tn, T h, const T (&u)[n],
                                            const T (&un)[n], const T (&K)[6][n]) {
  while (js < a.k) {
    const T tau = __ldg(a.tau + js);
    if (!(tau <= tn)) break;
    if (tau == tn) {
      store_point<n>(a, i, js, un);
    } else {
      T o[n];
      rodas4_interp<n, T>((tau - t) / h, u, un, K, o);
      store_point<n>(a, i, js, o);
    }
    ++js;
  }
}

template <class M, class T, bool SAVE> struct Rodas4Lane {
  static constexpr int n = M::n;
  T u[n], par[M::m], F0[n];
  T t, h, lq_old;   // lq_old = log2 q_old (DESIGN R2)
  int32_t nacc, nrej, ret, js;
  int64_t attempts;
  bool done;

  __device__ __forceinline__ void init(const Args<T>& a, int64_t i) {
    load_column<M, T>(a, i, u, par);
    t = a.t0; h = a.dt0; lq_old = T(kLFloor);
    nacc = nrej = 0; ret = RET_SUCCESS; js = 0; attempts = 0; done = false;
    M::f(u, par, t, F0);
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
    }
    if (!all_finite<n>(F0)) { ret = RET_DIVERGED; done = true; }
    else if (!(t < a.tf)) done = true;
  }

  __device__ __forceinline__ void step(const Args<T>& a, int64_t i) {
    if (attempts >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
    const bool last = (t + h >= a.tf);
    if (last) h = a.tf - t;
    ++attempts;
    T un[n], K[6][n];
    if (!rodas4_step<M, T>(par, t, h, u, F0, un, K)) {
      h = h * T(0.5);                       // singular W: reject and halve (DESIGN R10)
      ++nrej;
      if (t + h == t) { ret = RET_SINGULAR; done = true; }
      return;
    }
    const T q2 = error_q2<n, T>(K[5], u, un, a.abstol, a.reltol);
    if (q2 < T(1)) {
      const T tn = last ? a.tf : t + h;
      if (SAVE) rodas4_save<n, T>(a, i, js, t, tn, h, u, un, K);
      t = tn;
#pragma unroll (n <= 8 ? n : 1)
      for (int j = 0; j < n; ++j) u[j] = un[j];
      M::f(u, par, t, F0);
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, 7.0 / 40.0, 2.0 / 20.0);
    } else {
      h = pi_reject<T>(h, q2, 7.0 / 40.0);
      ++nrej;
    }
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  __device__ __forceinline__ void finish(const Args<T>& a, int64_t i) {
    if (SAVE) {
      T nanv[n];
#pragma unroll (n <= 8 ? n : 1)
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

// Fixed-step Rodas4 on the DESIGN R3 grid; a singular W ends the trajectory
// with RET_SINGULAR.
template <class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) rodas4_fixed_kernel(const Args<T> a) {
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
      const T tn = last ? a.tf : (T)(a.t0d + (double)(s + 1) * a.dtd);
      T un[n], K[6][n];
      if (!rodas4_step<M, T>(par, t, h, u, F0, un, K)) { ret = RET_SINGULAR; break; }
      if (SAVE) rodas4_save<n, T>(a, i, js, t, tn, h, u, un, K);
#pragma unroll (n <= 8 ? n : 1)
      for (int j = 0; j < n; ++j) u[j] = un[j];
      if (!last) M::f(u, par, tn, F0);
      ++nacc;
    }
    if (ret == RET_SUCCESS && !all_finite<n>(u)) ret = RET_DIVERGED;
  }
  if (SAVE) {
    T nanv[n];
#pragma unroll (n <= 8 ? n : 1)
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
