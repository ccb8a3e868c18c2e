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
  template <class T> __device__ __forceinline__ static void f(const T (&y)[3], const T (&p)[m], T, T (&o)[3]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) o[j] = p[0] * y[j];
  }
  template <class T> __device__ __forceinline__ static void g(const T (&y)[3], const T (&p)[m], T, T (&b)[3]) {
#pragma unroll
    for (int j = 0; j < 3; ++j) b[j] = p[1] * y[j];
  }
};

struct ExpDecay {  // u' = −λu
  static constexpr int n = 1, m = 1, nw = 0;
  template <class T> __device__ __forceinline__ static void f(const T (&y)[1], const T (&p)[1], T, T (&o)[1]) {
    o[0] = (-p[0]) * y[0];
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&)[1], const T (&p)[1], T, T (&J)[1][1]) {
    J[0][0] = -p[0];
  }
};

struct Harmonic {  // x' = v, v' = −ω²x
  static constexpr int n = 2, m = 1, nw = 0;
  template <class T> __device__ __forceinline__ static void f(const T (&y)[2], const T (&p)[1], T, T (&o)[2]) {
    o[0] = y[1];
    o[1] = -(p[0] * y[0]);
  }
  template <class T> __device__ __forceinline__ static void jac(const T (&y)[2], const T (&p)[1], T, T (&J)[2][2]) {
    J[0][0] = T(0); J[0][1] = T(1); J[1][0] = -p[0]; J[1][1] = T(0);
  }
};

}  // namespace ens
