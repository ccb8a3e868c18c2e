// vec2.cuh — f2: two fp32 lanes per thread on sm_100's packed FP32 path
// (FFMA2 / FADD2 / FMUL2). Each component is rounded exactly like the scalar
// __fmaf_rn / __fadd_rn / __fmul_rn, so a thread carrying two trajectories in
// f2 computes bit-for-bit what two scalar threads would — with half the issue
// slots, which is what the FP32-issue-bound Tsit5 kernel needs.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace ens {

struct f2 {
  float2 v;
  __device__ __forceinline__ f2() {}
  __device__ __forceinline__ f2(float2 x) : v(x) {}
  __device__ __forceinline__ f2(float a, float b) : v(make_float2(a, b)) {}
  // broadcast of a constant: T(double) rounds the double once to float, as in the scalar path
  __device__ __forceinline__ explicit f2(double x) : v(make_float2((float)x, (float)x)) {}
  __device__ __forceinline__ explicit f2(float x) : v(make_float2(x, x)) {}
  __device__ __forceinline__ explicit f2(int x) : v(make_float2((float)x, (float)x)) {}
};

__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return f2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator-(f2 a) { return f2(make_float2(-a.v.x, -a.v.y)); }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) { return f2(__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))); }
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return f2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator/(f2 a, f2 b) { return f2(a.v.x / b.v.x, a.v.y / b.v.y); }   // IEEE, per lane
template <> __device__ __forceinline__ f2 fmaT<f2>(f2 a, f2 b, f2 c) { return f2(__ffma2_rn(a.v, b.v, c.v)); }

// Scalar type of a lane vector and how many trajectories one thread carries.
template <class V> struct LaneOf { using T = V; static constexpr int W = 1; };
template <> struct LaneOf<f2> { using T = float; static constexpr int W = 2; };

template <class V> __device__ __forceinline__ typename LaneOf<V>::T lane(const V& x, int) { return x; }
__device__ __forceinline__ float lane(const f2& x, int w) { return w ? x.v.y : x.v.x; }
template <class V> __device__ __forceinline__ V make_lanes(typename LaneOf<V>::T a, typename LaneOf<V>::T) {
  return a;
}
template <> __device__ __forceinline__ f2 make_lanes<f2>(float a, float b) { return f2(a, b); }
template <class V> __device__ __forceinline__ V splat(typename LaneOf<V>::T a) { return make_lanes<V>(a, a); }

// ------------------------------------------------ packed R2 polynomials --
// log2 of DESIGN R2 on both lanes (Box–Muller radii, R8): the same operations
// per lane as log2_spec<float>, the polynomial and the quotient refinement as FFMA2.
// log2_quot on both lanes: two reciprocals, the refinement as FFMA2 (same
// per-lane rounding as the scalar sequence).
__device__ __forceinline__ f2 log2_quot2(f2 m) {
  const f2 a = m - f2(1.0f), b = m + f2(1.0f), nb = -b;
  f2 r(rcp_approx(b.v.x), rcp_approx(b.v.y));
  r = fmaT(r, fmaT(nb, r, f2(1.0f)), r);
  const f2 q = fmaT(a, r, f2(0.0f));
  return fmaT(r, fmaT(nb, q, a), q);
}
__device__ __forceinline__ f2 log2_spec2(float x0, float x1) {
  int e0, e1;
  float m0 = frexpT(x0, &e0), m1 = frexpT(x1, &e1);
  if (m0 < float(0.70710678118654752440)) { m0 = m0 * 2.0f; e0 -= 1; }
  if (m1 < float(0.70710678118654752440)) { m1 = m1 * 2.0f; e1 -= 1; }
  const f2 m(m0, m1);
  const f2 sv = log2_quot2(m);
  const f2 s2 = sv * sv;
  f2 acc = f2(pw_lc(PwDeg<float>::L));
#pragma unroll
  for (int k = PwDeg<float>::L - 1; k >= 0; --k) acc = fmaT(s2, acc, f2(pw_lc(k)));
  return fmaT(sv, acc, f2((float)e0, (float)e1));
}
}  // namespace ens
