// verner_launch.cuh — launch templates shared by k_vern7.cu and k_vern9.cu
// (one translation unit per tableau keeps the parallel build balanced).
#pragma once
#include "launch.cuh"
#include "verner.cuh"

namespace ens {

template <class Tab, class M, class T>
ens_status run_verner(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    if (save) launch_fixed(verner_fixed_kernel<Tab, M, T, true>, a, s);
    else launch_fixed(verner_fixed_kernel<Tab, M, T, false>, a, s);
  } else {
    // fp64 Vern9 holds ~138 registers: capped at 128 (two 256-thread blocks per SM) it keeps
    // 16 warps resident instead of 12 (1.76 -> 1.67 ms on the tight-tolerance config)
    if (sizeof(T) == 8 && Tab::S == 16 && M::n <= 4) {
      if (save) launch_adaptive<VernerLane<Tab, M, T, true>, T, 2>(a, opt->refill, s);
      else launch_adaptive<VernerLane<Tab, M, T, false>, T, 2>(a, opt->refill, s);
    } else {
      if (save) launch_adaptive<VernerLane<Tab, M, T, true>, T>(a, opt->refill, s);
      else launch_adaptive<VernerLane<Tab, M, T, false>, T>(a, opt->refill, s);
    }
  }
  return launch_status();
}

template <class Tab, class T>
ens_status launch_verner_tab(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return with_ode_model(model, [&](auto mt) -> ens_status {
    using M = decltype(mt);
    if constexpr (HasEvent<M>::value || M::n > 8) return ENS_E_UNSUPPORTED;   // events: Tsit5; n = 20: stiff only
    else return run_verner<Tab, M, T>(a, opt, s);
  });
}

}  // namespace ens
