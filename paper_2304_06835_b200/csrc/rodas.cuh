// rodas.cuh — per-thread W-form Rosenbrock integrators for sm_100a:
// Rodas4 (GPURodas4; DESIGN R20), Rodas5 (DESIGN R22) and its
// re-optimisation Rodas5P (GPURodas5P; DESIGN R23). NEXT-2.
//
// One exact Jacobian per step (analytic or in-kernel forward AD), one
// in-register LU of W = I/(hγ) − J, S triangular solves and S RHS evaluations
// (S = 6 / 8); stiffly accurate, so the error estimate is the last stage k_S.
// Like Rosenbrock23 there is no Newton iteration. All stage
// vectors, J, W and its LU stay in registers for n ≤ 8. Rodas4 saves through
// its dense output; Rodas5 / Rodas5P (their dense-output coefficients are not
// recoverable offline) store at a save point one step of the method from the
// step's start (R24), so the step sequence does not depend on saveat.
#pragma once
#include "common.cuh"
#include "models_stiff.cuh"
#include "ros23.cuh"   // lu_factor / lu_solve

namespace ens {

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
__host__ __device__ constexpr double rd5_a(int s, int j) {
  constexpr double A[8][7] = {
      {0, 0, 0, 0, 0, 0, 0},
      {2.0, 0, 0, 0, 0, 0, 0},
      {3.040894194418781, 1.041747909077569, 0, 0, 0, 0, 0},
      {2.576417536461461, 1.622083060776640, -0.9089668560264532, 0, 0, 0, 0},
      {2.760842080225597, 1.446624659844071, -0.3036980084553738, 0.2877498600325443, 0, 0, 0},
      {-14.09640773051259, 6.925207756232704, -41.47510893210728, 2.343771018586405, 24.13215229196062, 0, 0},
      {-14.09640773051259, 6.925207756232704, -41.47510893210728, 2.343771018586405, 24.13215229196062, 1.0, 0},
      {-14.09640773051259, 6.925207756232704, -41.47510893210728, 2.343771018586405, 24.13215229196062, 1.0,
       1.0}};
  return A[s][j];
}
__host__ __device__ constexpr double rd5_c(int s, int j) {
  constexpr double C[8][7] = {
      {0, 0, 0, 0, 0, 0, 0},
      {-10.31323885133993, 0, 0, 0, 0, 0, 0},
      {-21.04823117650003, -7.234992135176716, 0, 0, 0, 0, 0},
      {32.22751541853323, -4.943732386540191, 19.44922031041879, 0, 0, 0, 0},
      {-20.69865579590063, -8.816374604402768, 1.260436877740897, -0.7495647613787146, 0, 0, 0},
      {-46.22004352711257, -17.49534862857472, -289.6389582892057, 93.60855400400906, 318.3822534212147, 0, 0},
      {34.20013733472935, -14.15535402717690, 57.82335640988400, 25.83362985412365, 1.408950972071624,
       -6.551835421242162, 0},
      {42.57076742291101, -13.80770672017997, 93.98938432427124, 18.77919633714503, -31.58359187223370,
       -6.685968952921985, -5.810979938412932}};
  return C[s][j];
}

// Rodas5P (Steinebach's re-optimisation of Rodas5; GPURodas5P; DESIGN R23):
// same stage structure (Y7 = Y6 + k6, Y8 = Y7 + k7), γ = 0.21193756319429014.
__host__ __device__ constexpr double rd5p_a(int s, int j) {
  constexpr double A[8][7] = {
      {0, 0, 0, 0, 0, 0, 0},
      {3.0, 0, 0, 0, 0, 0, 0},
      {2.849394379747939, 0.45842242204463923, 0, 0, 0, 0, 0},
      {-6.954028509809101, 2.489845061869568, -10.358996098473584, 0, 0, 0, 0},
      {2.8029986275628964, 0.5072464736228206, -0.3988312541770524, -0.04721187230404641, 0, 0, 0},
      {-7.502846399306121, 2.561846144803919, -11.627539656261098, -0.18268767659942256, 0.030198172008377946, 0,
       0},
      {-7.502846399306121, 2.561846144803919, -11.627539656261098, -0.18268767659942256, 0.030198172008377946, 1.0,
       0},
      {-7.502846399306121, 2.561846144803919, -11.627539656261098, -0.18268767659942256, 0.030198172008377946, 1.0,
       1.0}};
  return A[s][j];
}
__host__ __device__ constexpr double rd5p_c(int s, int j) {
  constexpr double C[8][7] = {
      {0, 0, 0, 0, 0, 0, 0},
      {-14.155112264123755, 0, 0, 0, 0, 0, 0},
      {-17.97296035885952, -2.859693295451294, 0, 0, 0, 0, 0},
      {147.12150275711716, -1.41221402718213, 71.68940251302358, 0, 0, 0, 0},
      {165.43517024871676, -0.4592823456491126, 42.90938336958603, -5.961986721573306, 0, 0, 0},
      {24.854864614690072, -3.0009227002832186, 47.4931110020768, 5.5814197821558125, -0.6610691825249471, 0, 0},
      {30.91273214028599, -3.1208243349937974, 77.79954646070892, 34.28646028294783, -19.097331116725623,
       -28.087943162872662, 0},
      {37.80277123390563, -3.2571969029072276, 112.26918849496327, 66.9347231244047, -40.06618937091002,
       -54.66780262877968, -9.48861652309627}};
  return C[s][j];
}

// Tableau traits: S stages, γ, W-form a / c, PI exponents (R2 rule, p = order).
struct Rodas4Tab {
  static constexpr int S = 6;
  static constexpr double gamma = 0.25, beta1 = 7.0 / 40.0, beta2 = 2.0 / 20.0;
  __host__ __device__ static constexpr double a(int s, int j) { return rd_a(s, j); }
  __host__ __device__ static constexpr double c(int s, int j) { return rd_c(s, j); }
};
struct Rodas5Tab {
  static constexpr int S = 8;
  static constexpr double gamma = 0.19, beta1 = 7.0 / 50.0, beta2 = 2.0 / 25.0;
  __host__ __device__ static constexpr double a(int s, int j) { return rd5_a(s, j); }
  __host__ __device__ static constexpr double c(int s, int j) { return rd5_c(s, j); }
};
struct Rodas5PTab {
  static constexpr int S = 8;
  static constexpr double gamma = 0.21193756319429014, beta1 = 7.0 / 50.0, beta2 = 2.0 / 25.0;
  __host__ __device__ static constexpr double a(int s, int j) { return rd5p_a(s, j); }
  __host__ __device__ static constexpr double c(int s, int j) { return rd5p_c(s, j); }
};

__host__ __device__ constexpr double rd_d(int r, int j) {   // r = 0: D2 (s1), r = 1: D3 (s2)
  constexpr double D[2][5] = {
      {10.12623508344586, -7.487995877610167, -34.80091861555747, -7.992771707568823, 1.025137723295662},
      {-0.6762803392801253, 6.087714651680015, 16.43084320892478, 24.76722511418386, -6.594389125716872}};
  return D[r][j];
}

// One W-form Rosenbrock step of tableau Tab (autonomous models). F0 = f(u).
// Outputs u_new and K = k1..k_S (E = k_S). Returns false if W is singular (the
// outputs are then meaningless).
template <class Tab, class M, class T>
__device__ __forceinline__ bool rodas_step(const T (&par)[M::m], T t, T h, const T (&u)[M::n],
                                           const T (&F0)[M::n], T (&un)[M::n], T (&K)[Tab::S][M::n]) {
  ENS_REQUIRE_AUTONOMOUS(M, "Rodas (no γ_i·h·∂f/∂t terms, P:125-136)");
  constexpr int n = M::n, S = Tab::S;
  T W[n][n];
  const T hg = h * T(Tab::gamma);
  const T ihg = T(1) / hg;
  const T ih = T(1) / h;
  int piv[n];
  T inv[n];
  bool pm;
  const bool ok = lu_factor_fast<M, n, T>(W, piv, inv, pm, [&](T (&A)[n][n]) {
    model_jacobian<M, T>(u, par, t, A);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int i = 0; i < n; ++i)
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) A[i][j] = (i == j ? ihg : T(0)) - A[i][j];   // W = I/(hγ) − J
  });
  lu_solve_w<n, T>(W, piv, inv, pm, F0, K[0]);                               // k1 = W⁻¹ f(u)
  T y[n], F[n], r[n];
#pragma unroll
  for (int s = 1; s < S; ++s) {
    T hc[S - 1];
#pragma unroll
    for (int j = 0; j < s; ++j) hc[j] = T(Tab::c(s, j)) * ih;                // c_sj / h
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int c = 0; c < n; ++c) {
      T acc = u[c];
#pragma unroll
      for (int j = 0; j < s; ++j) acc = fmaT(T(Tab::a(s, j)), K[j][c], acc);  // Y_s = u + Σ a_sj k_j
      y[c] = acc;
    }
    M::f(y, par, t, F);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int c = 0; c < n; ++c) {
      T acc = F[c];
#pragma unroll
      for (int j = 0; j < s; ++j) acc = fmaT(hc[j], K[j][c], acc);          // f(Y_s) + Σ (c_sj/h) k_j
      r[c] = acc;
    }
    lu_solve_w<n, T>(W, piv, inv, pm, r, K[s]);
  }
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
  for (int c = 0; c < n; ++c) un[c] = y[c] + K[S - 1][c];                    // u_new = Y_S + k_S
  return ok;
}

// RODAS continuous extension: (1−θ)u + θ(u_new + (1−θ)(s1 + θ s2)).
template <int n, class T>
__device__ __forceinline__ void rodas4_interp(T theta, const T (&u)[n], const T (&un)[n], const T (&K)[6][n],
                                              T (&o)[n]) {
  const T th1 = T(1) - theta;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
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
    T un[n], K[6][n];
    if (!rodas_step<Rodas4Tab, M, T>(par, t, h, u, F0, un, K)) {
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
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) u[j] = un[j];
      M::f(u, par, t, F0);
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, Rodas4Tab::beta1, Rodas4Tab::beta2);
    } else {
      h = pi_reject<T>(h, q2, Rodas4Tab::beta1);
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
      if (!rodas_step<Rodas4Tab, M, T>(par, t, h, u, F0, un, K)) { ret = RET_SINGULAR; break; }
      if (SAVE) rodas4_save<n, T>(a, i, js, t, tn, h, u, un, K);
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) u[j] = un[j];
      if (!last) M::f(u, par, tn, F0);
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

// Rodas5 / Rodas5P (R22, R23): adaptive lane with the R24 dense output, and a
// fixed-step kernel saving by the fixed-step save codes.
template <class Tab, class M, class T, bool SAVE> struct RodasSubLane {
  // Dense output (DESIGN R24): a save point τ inside an accepted step [t, tp]
  // stores one Rodas step from (t, u) of length τ − t (its own W = I − (τ − t)γJ
  // and LU; NaN if that W is singular). One call per attempted step or per such
  // save point, through one rodas_step call site (a second inlined copy doubled
  // the build time of the POLLU units); the same operations in the same order as
  // storing the saves inside the accepting call.
  static constexpr int n = M::n;
  T u[n], par[M::m], F0[n];
  T t, h, lq_old;
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

  __device__ __forceinline__ void accept_end(const Args<T>& a, int64_t i) {
    if (SAVE) {   // τ = tp stores u_new
      while (js < a.k && __ldg(a.tau + js) <= tp) { store_point<n>(a, i, js, up); ++js; }
    }
    pend = false;
    t = tp;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
    for (int j = 0; j < n; ++j) u[j] = up[j];
    M::f(u, par, t, F0);
    if (!(t < a.tf)) done = true;
    else if (t + h == t) { ret = RET_DTMIN; done = true; }
  }

  // n ≤ 4: the dense-output steps inside the accepting call (a second inlined copy of the
  // stage code; 4 % faster on C3, profiles/ab_r02/ab_r24_sites_r02z3.jsonl — cheap to build)
  static constexpr bool kInlineSaves = (n <= 4);
  __device__ __forceinline__ void step(const Args<T>& a, int64_t i) {
    if constexpr (kInlineSaves) step_inline(a, i);
    else step_one_site(a, i);
  }

  __device__ __forceinline__ void step_one_site(const Args<T>& a, int64_t i) {
    const bool sub = SAVE && pend;
    bool last = false;
    if (!sub) {
      if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
      last = (t + h >= a.tf);
      if (last) h = a.tf - t;
    }
    const T hs = sub ? __ldg(a.tau + js) - t : h;
    T y[n], K[Tab::S][n];
    const bool ok = rodas_step<Tab, M, T>(par, t, hs, u, F0, y, K);
    if (sub) {
      if (!ok) {
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
        for (int j = 0; j < n; ++j) y[j] = nanT<T>();
      }
      store_point<n>(a, i, js, y);
      ++js;
      if (!(js < a.k && __ldg(a.tau + js) < tp)) accept_end(a, i);
      return;
    }
    if (!ok) {
      h = h * T(0.5);                       // singular W: reject and halve (DESIGN R10)
      ++nrej;
      if (t + h == t) { ret = RET_SINGULAR; done = true; }
      return;
    }
    const T q2 = error_q2<n, T>(K[Tab::S - 1], u, y, a.abstol, a.reltol);
    if (q2 < T(1)) {
      tp = last ? a.tf : t + h;
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) up[j] = y[j];
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

  __device__ __forceinline__ void step_inline(const Args<T>& a, int64_t i) {
    if (nacc + nrej >= a.max_steps) { ret = RET_MAXITERS; done = true; return; }
    const bool last = (t + h >= a.tf);
    if (last) h = a.tf - t;
    T un[n], K[Tab::S][n];
    if (!rodas_step<Tab, M, T>(par, t, h, u, F0, un, K)) {
      h = h * T(0.5);                       // singular W: reject and halve (DESIGN R10)
      ++nrej;
      if (t + h == t) { ret = RET_SINGULAR; done = true; }
      return;
    }
    const T q2 = error_q2<n, T>(K[Tab::S - 1], u, un, a.abstol, a.reltol);
    if (q2 < T(1)) {
      const T tn = last ? a.tf : t + h;
      if (SAVE) {
        while (js < a.k) {
          const T tau = __ldg(a.tau + js);
          if (!(tau <= tn)) break;
          if (tau == tn) {
            store_point<n>(a, i, js, un);
          } else {
            T o[n];
            if (!rodas_step<Tab, M, T>(par, t, tau - t, u, F0, o, K)) {
#pragma unroll
              for (int j = 0; j < n; ++j) o[j] = nanT<T>();
            }
            store_point<n>(a, i, js, o);
          }
          ++js;
        }
      }
      t = tn;
#pragma unroll
      for (int j = 0; j < n; ++j) u[j] = un[j];
      M::f(u, par, t, F0);
      ++nacc;
      h = pi_accept<T>(h, q2, lq_old, Tab::beta1, Tab::beta2);
    } else {
      h = pi_reject<T>(h, q2, Tab::beta1);
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

template <class Tab, class M, class T, bool SAVE>
__global__ void __launch_bounds__(256) rodas_coded_fixed_kernel(const Args<T> a) {
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
      T un[n], K[Tab::S][n];
      // fixed-step save codes (verner_fixed_kernel): the step's interior save points first (R24
      // steps of length τ − t from (t, u); NaN if that W is singular), then the step — one call site
      bool ok;
      const int js0 = js;
      for (;;) {
        bool sub = false;
        T hs = h;
        if (SAVE && js < a.k) {
          const int64_t code = __ldg(a.save_step + js);
          if ((code >> 1) == s + 1 && (code & 1)) { sub = true; hs = __ldg(a.tau + js) - t; }
        }
        ok = rodas_step<Tab, M, T>(par, t, hs, u, F0, un, K);
        if (!sub) break;
        if (!ok) {
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
          for (int j = 0; j < n; ++j) un[j] = nanT<T>();
        }
        store_point<n>(a, i, js, un);
        ++js;
      }
      if (!ok) { js = js0; ret = RET_SINGULAR; break; }   // the step failed: its save points stay unreached (NaN)
      if (SAVE) {   // τ = t_{s+1}
        while (js < a.k && __ldg(a.save_step + js) == ((s + 1) << 1)) { store_point<n>(a, i, js, un); ++js; }
      }
#pragma unroll (n <= kUnrollMax ? n : kPartialUnroll)
      for (int j = 0; j < n; ++j) u[j] = un[j];
      if (!last) M::f(u, par, (T)(a.t0d + (double)(s + 1) * a.dtd), F0);
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
