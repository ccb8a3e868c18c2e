// verner.cuh — per-thread Verner explicit integrators for sm_100a: Vern7
// (10-stage 7(6)) and Vern9 (16-stage 9(8)) — GPUVern7 / GPUVern9,
// P:319-320; NEXT-1; DESIGN R21.
//
// Verner's pairs; the embedded weights are derived from the order conditions
// (R21). All stage vectors stay in registers;
// zero tableau entries are compile-time constants, so their terms vanish from
// the instruction stream. Dense output (R24): a save point inside an accepted
// step stores one step of the same method from the step's start to the save
// point, so every saved value carries the method's order and the step
// sequence does not depend on saveat.
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
  constexpr double BT[10] = {0.0025470118799321617, 0, 0, -0.0096583948727968315, 0.042064709756393717,
                             -0.066682243746923789, 0.26500974646212530, -0.29430311714032503,
                             0.081317472324950901, -0.020295184663356433};
  return BT[j];
}

__host__ __device__ constexpr double v9_a(int s, int j) {
  constexpr double A[16][15] = {
      {0},
      {0.03462},
      {-0.0389335438857287, 0.13595789452451916},
      {0.03638413148954267, 0, 0.10915239446862801},
      {2.0257639143939694, 0, -7.638023836496292, 6.173259922102322},
      {0.05112275589406061, 0, 0, 0.17708237945550218, 0.0008027762409222536},
      {0.13160063579752163, 0, 0, -0.2957276252669636, 0.08781378035642955, 0.6213052975225274},
      {0.07166666666666667, 0, 0, 0, 0, 0.33055335789153195, 0.2427799754418014},
      {0.071806640625, 0, 0, 0, 0, 0.3294380283228177, 0.1165190029271823, -0.034013671875},
      {0.04836757646340646, 0, 0, 0, 0, 0.03928989925676164, 0.10547409458903446, -0.021438652846483126,
       -0.10412291746271944},
      {-0.026645614872014785, 0, 0, 0, 0, 0.03333333333333333, -0.1631072244872467, 0.03396081684127761,
       0.1572319413814626, 0.21522674780318796},
      {0.03689009248708622, 0, 0, 0, 0, -0.1465181576725543, 0.2242577768172024, 0.02294405717066073,
       -0.0035850052905728597, 0.08669223316444385, 0.43838406519683376},
      {-0.4866012215113341, 0, 0, 0, 0, -6.304602650282853, -0.2812456182894729, -2.679019236219849,
       0.5188156639241577, 1.3653531876033418, 5.8850910885039465, 2.8028087862720628},
      {0.4185367457753472, 0, 0, 0, 0, 6.724547581906459, -0.42544428016461133, 3.3432791530012653,
       0.6170816631175374, -0.9299661239399329, -6.099948804751011, -3.002206187889399, 0.2553202529443446},
      {-0.7793740861228848, 0, 0, 0, 0, -13.937342538107776, 1.2520488533793563, -14.691500408016868,
       -0.494705058533141, 2.2429749091462368, 13.367893803828643, 14.396650486650687, -0.79758133317768,
       0.4409353709534278},
      {2.0580513374668867, 0, 0, 0, 0, 22.357937727968032, 0.9094981099755646, 35.89110098240264,
       -3.442515027624454, -4.865481358036369, -18.909803813543427, -34.26354448030452, 1.2647565216956427}};
  return j < 15 ? A[s][j] : 0.0;
}
__host__ __device__ constexpr double v9_b(int j) {
  constexpr double B[16] = {0.014611976858423152, 0, 0, 0, 0, 0, 0, -0.3915211862331339, 0.23109325002895065,
                            0.12747667699928525, 0.2246434176204158, 0.5684352689748513, 0.058258715572158275,
                            0.13643174034822156, 0.030570139830827976, 0};
  return B[j];
}
__host__ __device__ constexpr double v9_bt(int j) {   // b − b̂ (R21)
  constexpr double BT[16] = {-0.0053579882904629451, 0, 0, 0, 0, 0, 0, -2.5830204911866472,
                             0.14252253154724535, 0.013420653512739405, -0.028672962914203417,
                             2.6249996552197984, -0.28255096432928784, 0.13643174034822156,
                             0.030570139830824279, -0.048342313738227605};
  return BT[j];
}

// Tableau traits: S stages, a / b / b̃, PI exponents (R2 rule with p = order).
struct Vern7Tab {
  static constexpr int S = 10;
  static constexpr double beta1 = 7.0 / 70.0, beta2 = 2.0 / 35.0;
  __host__ __device__ static constexpr double a(int s, int j) { return j < 9 ? v7_a(s, j) : 0.0; }
  __host__ __device__ static constexpr double b(int j) { return v7_b(j); }
  __host__ __device__ static constexpr double bt(int j) { return v7_bt(j); }
};
struct Vern9Tab {
  static constexpr int S = 16;
  static constexpr double beta1 = 7.0 / 90.0, beta2 = 2.0 / 45.0;
  __host__ __device__ static constexpr double a(int s, int j) { return v9_a(s, j); }
  __host__ __device__ static constexpr double b(int j) { return v9_b(j); }
  __host__ __device__ static constexpr double bt(int j) { return v9_bt(j); }
};

// K[0] = f(u) on entry; fills K[1..S−1], u_new and (if WANT_E) E = h·Σ b̃_j k_j.
template <class Tab, class M, class T, bool WANT_E>
__device__ __forceinline__ void verner_step(const T (&par)[M::m], T t, T h, const T (&u)[M::n],
                                            T (&K)[Tab::S][M::n], T (&un)[M::n], T (&E)[M::n]) {
  ENS_REQUIRE_AUTONOMOUS(M, "Vern7 / Vern9 (stages evaluated at the step start time)");
  constexpr int n = M::n, S = Tab::S;
#pragma unroll
  for (int s = 1; s < S; ++s) {
    T y[n];
#pragma unroll
    for (int c = 0; c < n; ++c) {
      T acc = u[c];
#pragma unroll
      for (int j = 0; j < s; ++j)
        if (Tab::a(s, j) != 0.0) acc = fmaT(h * T(Tab::a(s, j)), K[j][c], acc);
      y[c] = acc;
    }
    M::f(y, par, t, K[s]);
  }
#pragma unroll
  for (int c = 0; c < n; ++c) {
    T acc = u[c];
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (Tab::b(j) != 0.0) acc = fmaT(h * T(Tab::b(j)), K[j][c], acc);
    un[c] = acc;
    if (WANT_E) {
      T e = T(Tab::bt(0)) * K[0][c];
#pragma unroll
      for (int j = 1; j < S; ++j)
        if (Tab::bt(j) != 0.0) e = fmaT(T(Tab::bt(j)), K[j][c], e);
      E[c] = h * e;
    }
  }
}

// The lane: one attempted step per call. With saves, an accepted step whose
// interval holds interior save points is completed over several calls — one
// R24 dense-output step per call, through the same verner_step call site as the
// attempts, so the stage code is inlined once (a second inlined copy doubled the
// build time of these units). Same operations in the same order as storing the
// saves inside the accepting call.
template <class Tab, class M, class T, bool SAVE> struct VernerLane {
  static constexpr int n = M::n;
  T u[n], par[M::m], F0[n];
  T t, h, lq_old;   // lq_old = log2 q_old (DESIGN R2)
  int32_t nacc, nrej, ret, js;
  bool done;
  T up[n], tp;      // SAVE: the accepted step's end state and time while its interior saves are produced
  bool pend;

  __device__ __forceinline__ void init(const Args<T>& a, int64_t i) {
    load_column<M, T>(a, i, u, par);
    t = a.t0; h = a.dt0; lq_old = T(kLFloor);
    nacc = nrej = 0; ret = RET_SUCCESS; js = 0; done = false; pend = false;
    M::f(u, par, t, F0);
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= t) { store_point<n>(a, i, js, u); ++js; }
    }
    if (!all_finite<n>(F0)) { ret = RET_DIVERGED; done = true; }
    else if (!(t < a.tf)) done = true;
  }

  // end of an accepted step [t, tp]: a save point at τ = tp stores u_new; advance
  __device__ __forceinline__ void accept_end(const Args<T>& a, int64_t i) {
    if (SAVE) {
      while (js < a.k && __ldg(a.tau + js) <= tp) { store_point<n>(a, i, js, up); ++js; }
    }
    pend = false;
    t = tp;
#pragma unroll
    for (int c = 0; c < n; ++c) u[c] = up[c];
    M::f(u, par, t, F0);
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  __device__ __forceinline__ void step(const Args<T>& a, int64_t i) {
    const bool sub = SAVE && pend;   // an interior save point τ ∈ (t, tp) of the accepted step
    bool last = false;
    if (!sub) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
      last = (t + h >= a.tf);
      if (last) h = a.tf - t;
    }
    const T hs = sub ? __ldg(a.tau + js) - t : h;
    T K[Tab::S][n], y[n], E[n];
#pragma unroll
    for (int c = 0; c < n; ++c) K[0][c] = F0[c];
    verner_step<Tab, M, T, true>(par, t, hs, u, K, y, E);
    if (sub) {                        // R24: the step of length τ − t from (t, u)
      store_point<n>(a, i, js, y);
      ++js;
      if (!(js < a.k && __ldg(a.tau + js) < tp)) accept_end(a, i);
      return;
    }
    const T q2 = error_q2<n, T>(E, u, y, a.abstol, a.reltol);
    if (q2 < T(1)) {
      tp = last ? a.tf : t + h;
#pragma unroll
      for (int c = 0; c < n; ++c) up[c] = y[c];
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, Tab::beta1, Tab::beta2);
      if (SAVE && js < a.k && __ldg(a.tau + js) < tp) { pend = true; return; }
      accept_end(a, i);
    } else {
      h = pi_reject<T>(h, q2, Tab::beta1);
      ++nrej;
      if (t + h == t) { ret = RET_DTMIN; done = true; }   // t < tf here
    }
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

// Fixed-step Verner on the DESIGN R3 grid. Saves by the fixed-step save codes
// of tsit5_save_coded (api.cu fixed_save_codes): code (s << 1) | interp is
// stored during step s − 1 → s, u_s itself (interp = 0) or the dense output
// of R24 from the step's start (interp = 1); code 0 = saved at t0.
template <class Tab, class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) verner_fixed_kernel(const Args<T> a) {
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
      T K[Tab::S][n], un[n], E[n];
      // the step's interior save points first (R24 steps of length τ − t from (t, u)), then
      // the step itself — one verner_step call site
      for (;;) {
        bool sub = false;
        T hs = h;
        if (SAVE && js < a.k) {
          const int64_t code = __ldg(a.save_step + js);
          if ((code >> 1) == s + 1 && (code & 1)) { sub = true; hs = __ldg(a.tau + js) - t; }
        }
#pragma unroll
        for (int c = 0; c < n; ++c) K[0][c] = F0[c];
        verner_step<Tab, M, T, false>(par, t, hs, u, K, un, E);
        if (!sub) break;
        store_point<n>(a, i, js, un);
        ++js;
      }
      if (SAVE) {   // τ = t_{s+1}
        while (js < a.k && __ldg(a.save_step + js) == ((s + 1) << 1)) { store_point<n>(a, i, js, un); ++js; }
      }
#pragma unroll
      for (int c = 0; c < n; ++c) u[c] = un[c];
      if (!last) M::f(u, par, (T)(a.t0d + (double)(s + 1) * a.dtd), F0);
      ++nacc;
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
