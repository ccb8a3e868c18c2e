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
  } else if (opt->refill || M::n > 4) {
    // refill scheduler, and the larger systems (HIRES / POLLU: the lane form measured 3 % faster
    // on POLLU than the written-out loop)
    if (save) launch_adaptive<Ros23Lane<M, T, true>, T>(a, opt->refill, s);
    else launch_adaptive<Ros23Lane<M, T, false>, T>(a, opt->refill, s);
  } else if constexpr (M::n <= 4) {
    // Static mapping of small systems: the written-out loop kernel; fp64 at ≥ 2 blocks of 256
    // per SM (≤ 128 registers; a cap at 3 blocks / 80 registers spills and was slower with this
    // loop, 11.91 vs 11.75 ms) when the ensemble fills more than two blocks per SM.
    if (sizeof(T) == 8 && a.N > (int64_t)sm_count() * 2 * 256) {
      auto kern = save ? ros23_static_kernel<M, T, true, 2> : ros23_static_kernel<M, T, false, 2>;
      const dim3 b(occupancy_block(kern, a.N));
      kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
    } else {
      auto kern = save ? ros23_static_kernel<M, T, true, 1> : ros23_static_kernel<M, T, false, 1>;
      const dim3 b(occupancy_block(kern, a.N));
      kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
    }
  }
  return launch_status();
}

// POLLU (fp64) instances, compiled in k_ros23_pollu.cu.
ens_status run_ros23_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s);
inline ens_status run_ros23_pollu(const Args<float>&, const ens_options*, cudaStream_t) { return ENS_E_UNSUPPORTED; }

}  // namespace ens
