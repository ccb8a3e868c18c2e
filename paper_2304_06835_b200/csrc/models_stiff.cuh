// models_stiff.cuh — the paper's stiff test suite for Rosenbrock23:
// OREGO (n=3), HIRES (n=8), POLLU (n=20). Right-hand sides are written over a
// generic value type Y (T, or Dual<T,n> for the in-kernel forward-mode AD
// Jacobian, ad.cuh / P:329) with parameters of type P = T; operations are
// evaluated left to right exactly as printed in the paper, the
// oracle types the same expressions independently.
#pragma once
#include "ad.cuh"
#include "common.cuh"

namespace ens {

// Oregonator: p = (k1, k2, k3) = (77.27, 8.375e-6, 0.161), y0 = (1, 2, 3), t ∈ [0, 30]
struct Orego {
  static constexpr int n = 3, m = 3, nw = 0;
  static constexpr bool lu_fast_path = false;   // W needs row exchanges often (ros23.cuh lu_factor_fast)
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  static constexpr bool ad_jac = true;
  template <class Y, class P> __device__ __forceinline__ static void f(const Y (&y)[3], const P (&p)[3], P,
                                                                        Y (&o)[3]) {
    const Y inner = (P(1) - p[1] * y[0]) - y[1];            // 1 − k2 y1 − y2
    o[0] = p[0] * (y[1] + y[0] * inner);                    // k1 (y2 + y1 (1 − k2 y1 − y2)); R16: printed "−k1" is a typo
    o[1] = (y[2] - (P(1) + y[0]) * y[1]) / p[0];            // (y3 − (1 + y1) y2) / k1
    o[2] = p[2] * (y[0] - y[2]);                            // k3 (y1 − y3)
  }
};

// HIRES: p = (1.71, 0.43, 8.32, 0.0007, 8.75, 10.03, 0.035, 1.12, 1.745, 280, 0.69, 1.81)
struct Hires {
  static constexpr int n = 8, m = 12, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  static constexpr bool ad_jac = true;
  template <class Y, class P> __device__ __forceinline__ static void f(const Y (&y)[8], const P (&p)[12], P,
                                                                        Y (&o)[8]) {
    o[0] = ((-(p[0] * y[0]) + p[1] * y[1]) + p[2] * y[2]) + p[3];
    o[1] = p[0] * y[0] - p[4] * y[1];
    o[2] = (-(p[5] * y[2]) + p[1] * y[3]) + p[6] * y[4];
    o[3] = (p[2] * y[1] + p[0] * y[2]) - p[7] * y[3];
    o[4] = (-(p[8] * y[4]) + p[1] * y[5]) + p[1] * y[6];
    const Y r = (p[9] * y[5]) * y[7];                       // 280 y6 y8
    o[5] = (((-r + p[10] * y[3]) + p[0] * y[4]) - p[1] * y[5]) + p[10] * y[6];
    o[6] = r - p[11] * y[6];
    o[7] = -r + p[11] * y[6];
  }
};

// POLLU, P:779-833 (u9, u16 read as y9, y16): p = k1..k25, 25 reaction rates.
struct Pollu {
  static constexpr int n = 20, m = 25, nw = 0;
  static constexpr bool autonomous = true;   // f, J (and g) ignore t: ∂f/∂t = 0
  static constexpr bool ad_jac = true;
  template <class Y, class P> __device__ __forceinline__ static void f(const Y (&y)[20], const P (&k)[25], P,
                                                                        Y (&o)[20]) {
    const Y r1 = k[0] * y[0], r2 = (k[1] * y[1]) * y[3], r3 = (k[2] * y[4]) * y[1], r4 = k[3] * y[6];
    const Y r5 = k[4] * y[6], r6 = (k[5] * y[6]) * y[5], r7 = k[6] * y[8], r8 = (k[7] * y[8]) * y[5];
    const Y r9 = (k[8] * y[10]) * y[1], r10 = (k[9] * y[10]) * y[0], r11 = k[10] * y[12];
    const Y r12 = (k[11] * y[9]) * y[1], r13 = k[12] * y[13], r14 = (k[13] * y[0]) * y[5], r15 = k[14] * y[2];
    const Y r16 = k[15] * y[3], r17 = k[16] * y[3], r18 = k[17] * y[15], r19 = k[18] * y[15];
    const Y r20 = (k[19] * y[16]) * y[5], r21 = k[20] * y[18], r22 = k[21] * y[18], r23 = (k[22] * y[0]) * y[3];
    const Y r24 = (k[23] * y[18]) * y[0], r25 = k[24] * y[19];
    o[0] = (((((((((((-r1 - r10) - r14) - r23) - r24) + r2) + r3) + r9) + r11) + r12) + r22) + r25);
    o[1] = ((((-r2 - r3) - r9) - r12) + r1) + r21;
    o[2] = (((-r15 + r1) + r17) + r19) + r22;
    o[3] = (((-r2 - r16) - r17) - r23) + r15;
    o[4] = ((((-r3 + P(2) * r4) + r6) + r7) + r13) + r20;
    o[5] = ((((-r6 - r8) - r14) - r20) + r3) + P(2) * r18;
    o[6] = ((-r4 - r5) - r6) + r13;
    o[7] = ((r4 + r5) + r6) + r7;
    o[8] = -r7 - r8;
    o[9] = (-r12 + r7) + r9;
    o[10] = ((-r9 - r10) + r8) + r11;
    o[11] = r9;
    o[12] = -r11 + r10;
    o[13] = -r13 + r12;
    o[14] = r14;
    o[15] = (-r18 - r19) + r16;
    o[16] = -r20;
    o[17] = r20;
    o[18] = ((((-r21 - r22) - r24) + r23) + r25);
    o[19] = -r25 + r24;
  }
};

// Jacobian dispatch: hand-written functor, or forward-mode AD for ad_jac models.
template <class M, class = void> struct HasAdJac { static constexpr bool value = false; };
template <class M> struct HasAdJac<M, decltype((void)M::ad_jac)> { static constexpr bool value = M::ad_jac; };

template <class M, class T>
__device__ __forceinline__ void model_jacobian(const T (&u)[M::n], const T (&p)[M::m], T t, T (&J)[M::n][M::n]) {
  if constexpr (HasAdJac<M>::value) ad_jacobian<M, T>(u, p, t, J);
  else M::jac(u, p, t, J);
}

}  // namespace ens
