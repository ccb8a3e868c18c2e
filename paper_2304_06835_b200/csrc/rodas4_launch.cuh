// rodas4_launch.cuh — the launch template of rodas4 (shared by k_rodas4.cu and k_rodas4_pollu.cu,
// which holds the POLLU (n = 20) instances: fully unrolled, they are the
// slowest units to compile, so they build in parallel with the rest).
#pragma once
#include "launch.cuh"
#include "rodas.cuh"

namespace ens {

template <class M, class T>
ens_status run_rodas4(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    if (save) launch_fixed(rodas4_fixed_kernel<M, T, true>, a, s);
    else launch_fixed(rodas4_fixed_kernel<M, T, false>, a, s);
  } else {
    if (save) launch_adaptive<Rodas4Lane<M, T, true>, T>(a, opt->refill, s);
    else launch_adaptive<Rodas4Lane<M, T, false>, T>(a, opt->refill, s);
  }
  return launch_status();
}

// POLLU (fp64) instances, compiled in k_rodas4_pollu.cu.
ens_status run_rodas4_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s);
inline ens_status run_rodas4_pollu(const Args<float>&, const ens_options*, cudaStream_t) { return ENS_E_UNSUPPORTED; }

}  // namespace ens
