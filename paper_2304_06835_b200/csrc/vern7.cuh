// vern7.cuh — per-thread Vern7 explicit 7(6) integrator for sm_100a (GPUVern7,
// P:319-320; NEXT-1; DESIGN R21).
//
// Verner's 10-stage 7th-order pair; the embedded order-6 weights are derived
// from the order conditions (R21). All ten stage vectors stay in registers;
// zero tableau entries are compile-time constants, so their terms vanish from
// the instruction stream. Saves keep the full order (R21): fixed step — on
// grid points; adaptive — the step is clipped to land on the next save point.
#pragma once
#include "common.cuh"
#include "models.cuh"

namespace ens {

__host__ __device__ constexpr double v7_a(int s, int j) {
  constexpr double A[10][9] = {
      {0, 0, 0, 0, 0, 0, 0, 0, 0},
      {0.005, 0, 0, 0, 0, 0, 0, 0, 0},
      {-1.07679012345679, 1.185679012345679, 0, 0, 0, 0, 0, 0, 0},
      {0.04083333333333333, 0, 0.1225, 0, 0, 0, 0, 0, 0},
      {0.6389139236255726, 0, -2.455672638223657, 2.272258714598084, 0, 0, 0, 0, 0},
      {-2.6615773750187572, 0, 10.804513886456137, -8.3539146573962, 0.820487594956657, 0, 0, 0, 0},
      {6.067741434696772, 0, -24.711273635911088, 20.427517930788895, -1.9061579788166472, 1.006172249242068, 0,
       0, 0},
      {12.054670076253203, 0, -49.75478495046899, 41.142888638604674, -4.461760149974004, 2.042334822239175,
       -0.09834843665406107, 0, 0},
      {10.138146522881808, 0, -42.6411360317175, 35.76384003992257, -4.3480228403929075, 2.0098622683770357,
       0.3487490460338272, -0.27143900510483127, 0},
      {-45.030072034298676, 0, 187.3272437654589, -154.02882369350186, 18.56465306347536, -7.141809679295079,
       1.3088085781613787, 0, 0}};
  return A[s][j];
}
__host__ __device__ constexpr double v7_b(int j) {
  constexpr double B[10] = {0.04715561848627222, 0, 0, 0.25750564298434153, 0.2621665397741262,
                            0.15216092656738558, 0.4939969170032485, -0.29430311714032503, 0.08131747232495111, 0};
  return B[j];
}
__host__ __device__ constexpr double v7_bt(int j) {   // b − b̂ (R21)
  constexpr double BT[10] = {0.0030925885828119940, 0, 0, -0.011727248681971966, 0.051075082200004638,
                             -0.080965757291055731, 0.32177553732670404, -0.35734362573070983,
                             0.098735890663364916, -0.024642467069148059};
  return BT[j];
}

// K[0] = f(u) on entry; fills K[1..9], u_new and (if WANT_E) E = h·Σ b̃_j k_j.
template <class M, class T, bool WANT_E>
__device__ __forceinline__ void vern7_step(const T (&par)[M::m], T t, T h, const T (&u)[M::n], T (&K)[10][M::n],
                                           T (&un)[M::n], T (&E)[M::n]) {
  constexpr int n = M::n;
#pragma unroll
  for (int s = 1; s < 10; ++s) {
    T y[n];
#pragma unroll
    for (int c = 0; c < n; ++c) {
      T acc = u[c];
#pragma unroll
      for (int j = 0; j < s; ++j)
        if (v7_a(s, j) != 0.0) acc = fmaT(h * T(v7_a(s, j)), K[j][c], acc);
      y[c] = acc;
    }
    M::f(y, par, t, K[s]);
  }
#pragma unroll
  for (int c = 0; c < n; ++c) {
    T acc = u[c];
#pragma unroll
    for (int j = 0; j < 10; ++j)
      if (v7_b(j) != 0.0) acc = fmaT(h * T(v7_b(j)), K[j][c], acc);
    un[c] = acc;
    if (WANT_E) {
      T e = T(v7_bt(0)) * K[0][c];
#pragma unroll
      for (int j = 1; j < 10; ++j)
        if (v7_bt(j) != 0.0) e = fmaT(T(v7_bt(j)), K[j][c], e);
      E[c] = h * e;
    }
  }
}

template <class M, class T, bool SAVE> struct Vern7Lane {
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
    const T target = (SAVE && js < a.k) ? __ldg(a.tau + js) : a.tf;   // next save point or tf (R21)
    const bool clip = (t + h >= target);
    if (clip) h = target - t;
    T K[10][n], un[n], E[n];
#pragma unroll
    for (int c = 0; c < n; ++c) K[0][c] = F0[c];
    vern7_step<M, T, true>(par, t, h, u, K, un, E);
    const T q2 = error_q2<n, T>(E, u, un, a.abstol, a.reltol);
    ++attempts;
    if (q2 < T(1)) {
      t = clip ? target : t + h;
#pragma unroll
      for (int c = 0; c < n; ++c) u[c] = un[c];
      if (SAVE && clip && js < a.k) { store_point<n>(a, i, js, u); ++js; }
      M::f(u, par, t, F0);
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, 7.0 / 70.0, 2.0 / 35.0);
    } else {
      h = pi_reject<T>(h, q2, 7.0 / 70.0);
      ++nrej;
    }
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  __device__ __forceinline__ void finish(const Args<T>& a, int64_t i) {
    if (SAVE) {
      T nanv[n];
#pragma unroll
      for (int c = 0; c < n; ++c) nanv[c] = nanT<T>();
      for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
    } else {
      store_point<n>(a, i, 0, u);
    }
    if (a.retcode) a.retcode[i] = ret;
    if (a.nacc) a.nacc[i] = nacc;
    if (a.nrej) a.nrej[i] = nrej;
  }
};

// Fixed-step Vern7 on the DESIGN R3 grid; saves at grid indices a.save_step.
template <class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) vern7_fixed_kernel(const Args<T> a) {
  constexpr int n = M::n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  T u[n], par[M::m], F0[n];
  load_column<M, T>(a, i, u, par);
  M::f(u, par, a.t0, F0);
  int js = 0;
  if (SAVE) {
    while (js < a.k && __ldg(a.save_step + js) == 0) { store_point<n>(a, i, js, u); ++js; }
  }
  int32_t ret = RET_SUCCESS, nacc = 0;
  if (!all_finite<n>(F0)) ret = RET_DIVERGED;
  else {
    for (int64_t s = 0; s < a.nsteps; ++s) {
      const bool last = (s == a.nsteps - 1);
      const T h = last ? a.h_last : a.dt0;
      const T t = (T)(a.t0d + (double)s * a.dtd);
      T K[10][n], un[n], E[n];
#pragma unroll
      for (int c = 0; c < n; ++c) K[0][c] = F0[c];
      vern7_step<M, T, false>(par, t, h, u, K, un, E);
#pragma unroll
      for (int c = 0; c < n; ++c) u[c] = un[c];
      if (!last) M::f(u, par, (T)(a.t0d + (double)(s + 1) * a.dtd), F0);
      ++nacc;
      if (SAVE) {
        while (js < a.k && __ldg(a.save_step + js) == s + 1) { store_point<n>(a, i, js, u); ++js; }
      }
    }
    if (!all_finite<n>(u)) ret = RET_DIVERGED;
  }
  if (SAVE) {
    T nanv[n];
#pragma unroll
    for (int c = 0; c < n; ++c) nanv[c] = nanT<T>();
    for (; js < a.k; ++js) store_point<n>(a, i, js, nanv);
  } else {
    store_point<n>(a, i, 0, u);
  }
  if (a.retcode) a.retcode[i] = ret;
  if (a.nacc) a.nacc[i] = nacc;
  if (a.nrej) a.nrej[i] = 0;
}

}  // namespace ens
