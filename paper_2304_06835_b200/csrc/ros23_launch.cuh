// ros23_launch.cuh — the launch template of ros23 (shared by k_ros23.cu and k_ros23_pollu.cu,
// which holds the POLLU (n = 20) instances: fully unrolled, they are the
// slowest units to compile, so they build in parallel with the rest).
#pragma once
#include "launch.cuh"
#include "ros23.cuh"

namespace ens {

template <class M, class T>
ens_status run_ros23(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    if (save) launch_fixed(ros23_fixed_kernel<M, T, true>, a, s);
    else launch_fixed(ros23_fixed_kernel<M, T, false>, a, s);
  } else {
    // fp64 Rosenbrock23 is latency-bound at 2 blocks/SM (97 regs); capping registers for a
    // third resident block is 6 % faster on C3 (profiles/ros23_minb_r01.log) — for small systems
    // only: HIRES (n = 8) spills under the cap and runs 17 % slower (profiles/ros23_minb_models_r01.log).
    // A cap of 4 blocks (64 regs) spills on C3 as well and is slower.
    // (only when the ensemble fills more than two blocks per SM: a small ensemble — the stiff suite's
    //  8192 — gains no residency from the cap and pays for its spills, OREGO 9 % slower)
    if (sizeof(T) == 8 && M::n <= 4 && !opt->refill && a.N > (int64_t)sm_count() * 2 * 256) {
      if (save) launch_adaptive<Ros23Lane<M, T, true>, T, 3>(a, false, s);
      else launch_adaptive<Ros23Lane<M, T, false>, T, 3>(a, false, s);
    } else {
      if (save) launch_adaptive<Ros23Lane<M, T, true>, T>(a, opt->refill, s);
      else launch_adaptive<Ros23Lane<M, T, false>, T>(a, opt->refill, s);
    }
  }
  return launch_status();
}

// POLLU (fp64) instances, compiled in k_ros23_pollu.cu.
ens_status run_ros23_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s);
inline ens_status run_ros23_pollu(const Args<float>&, const ens_options*, cudaStream_t) { return ENS_E_UNSUPPORTED; }

}  // namespace ens
