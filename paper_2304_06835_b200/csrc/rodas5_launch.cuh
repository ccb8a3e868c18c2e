// rodas5_launch.cuh — the launch template of the 8-stage Rosenbrock methods Rodas5 and
// Rodas5P (shared by k_rodas5.cu / k_rodas5p.cu and k_rodas5_pollu.cu / k_rodas5p_pollu.cu, which
// hold the POLLU (n = 20) instances: fully unrolled, they are the slowest units to compile, so they
// build in parallel with the rest).
#pragma once
#include "launch.cuh"
#include "rodas.cuh"

namespace ens {

template <class Tab, class M, class T>
ens_status run_rodas_sub(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    if (save) launch_fixed(rodas_coded_fixed_kernel<Tab, M, T, true>, a, s);
    else launch_fixed(rodas_coded_fixed_kernel<Tab, M, T, false>, a, s);
  } else if (sizeof(T) == 8 && M::n <= 4 && LuFastPath<M>::value) {
    // fp64 small systems with the LU fast path: capped at 128 registers (two 256-thread blocks
    // per SM); uncapped the instance holds 130 and would drop to 12 resident warps (C3: 11.5 vs
    // 11.0 ms before the cap, 10.6 ms with it)
    if (save) launch_adaptive<RodasSubLane<Tab, M, T, true>, T, 2>(a, opt->refill, s);
    else launch_adaptive<RodasSubLane<Tab, M, T, false>, T, 2>(a, opt->refill, s);
  } else {
    if (save) launch_adaptive<RodasSubLane<Tab, M, T, true>, T>(a, opt->refill, s);
    else launch_adaptive<RodasSubLane<Tab, M, T, false>, T>(a, opt->refill, s);
  }
  return launch_status();
}

template <class M, class T>
ens_status run_rodas5(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return run_rodas_sub<Rodas5Tab, M, T>(a, opt, s);
}
template <class M, class T>
ens_status run_rodas5p(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return run_rodas_sub<Rodas5PTab, M, T>(a, opt, s);
}

// POLLU (fp64) instances, compiled in k_rodas5_pollu.cu / k_rodas5p_pollu.cu.
ens_status run_rodas5_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s);
inline ens_status run_rodas5_pollu(const Args<float>&, const ens_options*, cudaStream_t) { return ENS_E_UNSUPPORTED; }
ens_status run_rodas5p_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s);
inline ens_status run_rodas5p_pollu(const Args<float>&, const ens_options*, cudaStream_t) { return ENS_E_UNSUPPORTED; }

}  // namespace ens
