// ad.cuh — forward-mode automatic differentiation inside the kernel (P:329:
// "Integration of solvers is done with forward-mode automatic differentiation
// within a GPU kernel"): Dual<T, N> carries a value and N partials; a model's
// right-hand side written over a generic value type yields the exact Jacobian
// J[i][k] = ∂f_i/∂y_k in one evaluation with unit seeds (DESIGN R15).
//
// Rounding order of every operation is part of the specification,
// implemented independently in the oracle. Mixed operands (dual ∘ scalar
// constant or parameter) use the reduced formulas below.
#pragma once
#include "common.cuh"

namespace ens {

template <class T, int N> struct Dual {
  T v;
  T d[N];
};

#define ENS_DUAL_UNROLL _Pragma("unroll")

template <class T, int N> __device__ __forceinline__ Dual<T, N> operator+(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v + b.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = a.d[k] + b.d[k];
  return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator-(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v - b.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = a.d[k] - b.d[k];
  return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator-(const Dual<T, N>& a) {
  Dual<T, N> r; r.v = -a.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = -a.d[k];
  return r;
}
// (a·b)' = fma(a, b', a'·b)
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator*(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v * b.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = fmaT(a.v, b.d[k], a.d[k] * b.v);
  return r;
}
// scalar ∘ dual: the scalar has no partials
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator*(T s, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = s * b.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = s * b.d[k];
  return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator*(const Dual<T, N>& a, T s) {
  Dual<T, N> r; r.v = a.v * s;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * s;
  return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator/(const Dual<T, N>& a, T s) {
  Dual<T, N> r; r.v = a.v / s;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = a.d[k] / s;
  return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator+(const Dual<T, N>& a, T s) {
  Dual<T, N> r = a; r.v = a.v + s; return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator+(T s, const Dual<T, N>& b) {
  Dual<T, N> r = b; r.v = s + b.v; return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator-(const Dual<T, N>& a, T s) {
  Dual<T, N> r = a; r.v = a.v - s; return r;
}
template <class T, int N> __device__ __forceinline__ Dual<T, N> operator-(T s, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = s - b.v;
  ENS_DUAL_UNROLL for (int k = 0; k < N; ++k) r.d[k] = -b.d[k];
  return r;
}

// J[i][k] = ∂f_i/∂y_k. Every partial is computed by its own chain of the rules
// above, independent of the other partials, so the columns may be produced in
// passes of W seeds each (W = n: one evaluation with unit seeds) with identical
// results. Small systems take one pass; for n > 4 the n-wide duals of every
// intermediate overflow the register file (POLLU: 17.7 KB of local memory per
// thread), so the columns are formed in passes of kAdPass<n> seeds.
template <int n> constexpr int kAdPass = (n <= 4) ? n : 1;

template <class M, class T>
__device__ __forceinline__ void ad_jacobian(const T (&u)[M::n], const T (&p)[M::m], T t, T (&J)[M::n][M::n]) {
  constexpr int n = M::n, W = kAdPass<n>;
  static_assert(n % W == 0, "AD pass width must divide n");
#pragma unroll (n <= kUnrollMax ? n / W : 1)
  for (int k0 = 0; k0 < n; k0 += W) {
    Dual<T, W> y[n], o[n];
#pragma unroll (n <= kUnrollMax ? n : 1)
    for (int i = 0; i < n; ++i) {
      y[i].v = u[i];
#pragma unroll
      for (int c = 0; c < W; ++c) y[i].d[c] = (i == k0 + c) ? T(1) : T(0);
    }
    M::f(y, p, t, o);
#pragma unroll (n <= kUnrollMax ? n : 1)
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int c = 0; c < W; ++c) J[i][k0 + c] = o[i].d[c];
  }
}

}  // namespace ens
