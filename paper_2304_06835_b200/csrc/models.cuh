// models.cuh — per-model device functors (the analogue of the paper's
// model-specific kernel generation: every solver kernel is a
// template instantiated per model, so f and J inline into the integrator).
//
// Each model: n states, m parameters, nw Wiener processes; f(y,p,t) in the
// canonical operation order of DESIGN §4; exact analytic Jacobian for the
// Rosenbrock path (the paper derives J by in-kernel forward AD); the
// diagonal diffusion for SDE models. All autonomous (∂f/∂t = 0).
#pragma once
#include "common.cuh"

namespace ens {

struct Lorenz {   // σ(y2−y1), ρy1 − y2 − y1y3, y1y2 − βy3
  static constexpr int n = 3, m = 3, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[3], const T (&p)[m], T, T (&o)[3]) {
    o[0] = p[0] * (y[1] - y[0]);
    o[1] = fmaT(y[0], p[1] - y[2], -y[1]);
    o[2] = fmaT(y[0], y[1], -(p[2] * y[2]));
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&y)[3], const T (&p)[m], T, T (&J)[3][3]) {
    J[0][0] = -p[0];       J[0][1] = p[0]; J[0][2] = T(0);
    J[1][0] = p[1] - y[2]; J[1][1] = T(-1); J[1][2] = -y[0];
    J[2][0] = y[1];        J[2][1] = y[0]; J[2][2] = -p[2];
  }
};

struct Robertson {  // P:671-677 with (k1,k2,k3) = p
  static constexpr int n = 3, m = 3, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[3], const T (&p)[m], T, T (&o)[3]) {
    const T r3 = (p[2] * y[1]) * y[2];
    o[0] = fmaT(-p[0], y[0], r3);
    o[2] = (p[1] * y[1]) * y[1];
    o[1] = fmaT(p[0], y[0], -r3) - o[2];
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&y)[3], const T (&p)[m], T, T (&J)[3][3]) {
    const T a = p[2] * y[2], b = p[2] * y[1], c = (p[1] * y[1]) * T(2);
    J[0][0] = -p[0]; J[0][1] = a;        J[0][2] = b;
    J[1][0] = p[0];  J[1][1] = (-a) - c; J[1][2] = -b;
    J[2][0] = T(0);  J[2][1] = c;        J[2][2] = T(0);
  }
};

template <bool MUL> struct LorenzSDE {  // DESIGN R9: drift = Lorenz, b_j = s (add) or s·u_j (mul)
  static constexpr int n = 3, m = 4, nw = 3;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[3], const T (&p)[m], T, T (&o)[3]) {
    o[0] = p[0] * (y[1] - y[0]);
    o[1] = fmaT(y[0], p[1] - y[2], -y[1]);
    o[2] = fmaT(y[0], y[1], -(p[2] * y[2]));
  }
  template <class T> __device__ __forceinline__ static void g(const T (&y)[3], const T (&p)[m], T, T (&b)[3]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) b[j] = MUL ? p[3] * y[j] : p[3];
  }
};

struct GBM {  // dX = rX dt + VX dW (diagonal, 3 independent components)
  static constexpr int n = 3, m = 2, nw = 3;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[3], const T (&p)[m], T, T (&o)[3]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) o[j] = p[0] * y[j];
  }
  template <class T> __device__ __forceinline__ static void g(const T (&y)[3], const T (&p)[m], T, T (&b)[3]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) b[j] = p[1] * y[j];
  }
};

// Noise increment x += G(y) ΔW in the model's canonical order.
// Diagonal models: x_j = fma(b_j, ΔW_j, x_j).
template <class M, class T>
__device__ __forceinline__ void diag_noise(const T (&y)[M::n], const T (&p)[M::m], T t, const T (&dW)[M::nw],
                                           T (&x)[M::n]) {
  T b[M::n];
  M::g(y, p, t, b);
#pragma unroll
  for (int j = 0; j < M::n; ++j) x[j] = fmaT(b[j], dW[j], x[j]);
}

// σ-factor stress-response CRN as a chemical Langevin SDE:
// y = ([σ], [A1], [A2], [A3]), p = (S, D, τ, ν0, n, η), 8 Wiener processes.
//   d[σ]  = (ν0 + H − [σ]) dt + η√(ν0 + H) dW1 − η√[σ] dW2,  H = (S[σ])^n / ((S[σ])^n + (D[A3])^n + 1)
//   d[A_k] = ([A_{k−1}] − [A_k])/τ dt + η√([A_{k−1}]/τ) dW_{2k+1} − η√([A_k]/τ) dW_{2k+2}
// DESIGN R14: non-negative parts inside powers and square roots; x^n by the
// polynomial 2^{n·L(x)} of R2 (x ∈ [1e-30, 1e30], exponent clamped to ±120).
struct CRN {
  static constexpr int n = 4, m = 6, nw = 8;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static T hill_pow(T x, T e) {
    const T xc = minT(maxT(x, T(1e-30)), T(1e30));
    const T z = minT(maxT(e * log2_spec<T>(xc), T(-120)), T(120));
    return exp2_spec<T>(z);
  }
  template <class T> __device__ __forceinline__ static void terms(const T (&y)[4], const T (&p)[m], T& sp, T& a3p,
                                                                  T& hill, T& itau) {
    sp = maxT(y[0], T(0));
    a3p = maxT(y[3], T(0));
    const T a = hill_pow<T>(p[0] * sp, p[4]);
    const T b = hill_pow<T>(p[1] * a3p, p[4]);
    hill = a / ((a + b) + T(1));
    itau = T(1) / p[2];
  }
  template <class T> __device__ __forceinline__ static void f(const T (&y)[4], const T (&p)[m], T, T (&o)[4]) {
    T sp, a3p, hill, itau;
    terms<T>(y, p, sp, a3p, hill, itau);
    o[0] = (p[3] + hill) - y[0];
    o[1] = (y[0] - y[1]) * itau;
    o[2] = (y[1] - y[2]) * itau;
    o[3] = (y[2] - y[3]) * itau;
  }
  // row i carries columns 2i, 2i+1: x_i = fma(G_i,2i, ΔW_2i, x_i); x_i = fma(G_i,2i+1, ΔW_2i+1, x_i)
  template <class T> __device__ __forceinline__ static void noise(const T (&y)[4], const T (&p)[m], T,
                                                                  const T (&dW)[8], T (&x)[4]) {
    T sp, a3p, hill, itau;
    terms<T>(y, p, sp, a3p, hill, itau);
    const T eta = p[5];
    T G[8];
    G[0] = eta * sqrtT(maxT(p[3] + hill, T(0)));
    G[1] = -(eta * sqrtT(sp));
    const T r1 = eta * sqrtT(sp * itau), r2 = eta * sqrtT(maxT(y[1], T(0)) * itau);
    const T r3 = eta * sqrtT(maxT(y[2], T(0)) * itau), r4 = eta * sqrtT(a3p * itau);
    G[2] = r1; G[3] = -r2; G[4] = r2; G[5] = -r3; G[6] = r3; G[7] = -r4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = fmaT(G[2 * i], dW[2 * i], x[i]);
      x[i] = fmaT(G[2 * i + 1], dW[2 * i + 1], x[i]);
    }
  }
};

// Bouncing ball with an event: x' = v, v' = −g; the
// condition g(u) = x (u[1] in the paper's 1-based Listing) crossing zero
// downward triggers the affect v ← −e·v; p = (g, e) (DESIGN R18).
struct Ball {
  static constexpr int n = 2, m = 2, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  static constexpr bool has_event = true;
  template <class T> __device__ __forceinline__ static void f(const T (&y)[2], const T (&p)[2], T, T (&o)[2]) {
    o[0] = y[1];
    o[1] = -p[0];
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&)[2], const T (&)[2], T, T (&J)[2][2]) {
    J[0][0] = T(0); J[0][1] = T(1); J[1][0] = T(0); J[1][1] = T(0);
  }
  template <class T> __device__ __forceinline__ static T event_g(const T (&y)[2]) { return y[0]; }
  template <class T> __device__ __forceinline__ static void affect(T (&y)[2], const T (&p)[2]) {
    y[1] = -(p[1] * y[1]);
  }
};
template <class M, class = void> struct HasEvent { static constexpr bool value = false; };
template <class M> struct HasEvent<M, decltype((void)M::has_event)> { static constexpr bool value = M::has_event; };

template <class M, class T>
__device__ __forceinline__ void apply_noise(const T (&y)[M::n], const T (&p)[M::m], T t, const T (&dW)[M::nw],
                                            T (&x)[M::n]) {
  if constexpr (M::nw == 8) M::noise(y, p, t, dW, x);
  else diag_noise<M, T>(y, p, t, dW, x);
}

struct ExpDecay {  // u' = −λu
  static constexpr int n = 1, m = 1, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[1], const T (&p)[1], T, T (&o)[1]) {
    o[0] = (-p[0]) * y[0];
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&)[1], const T (&p)[1], T, T (&J)[1][1]) {
    J[0][0] = -p[0];
  }
};

struct Harmonic {  // x' = v, v' = −ω²x
  static constexpr int n = 2, m = 1, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  template <class T> __device__ __forceinline__ static void f(const T (&y)[2], const T (&p)[1], T, T (&o)[2]) {
    o[0] = y[1];
    o[1] = -(p[0] * y[0]);
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&y)[2], const T (&p)[1], T, T (&J)[2][2]) {
    J[0][0] = T(0); J[0][1] = T(1); J[1][0] = -p[0]; J[1][1] = T(0);
  }
};

}  // namespace ens
