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

}  // namespace ens
