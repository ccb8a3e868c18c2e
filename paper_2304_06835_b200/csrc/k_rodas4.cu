// k_rodas4.cu — Rodas4 kernel instances (fixed step; adaptive static or
// refill) for the ODE models without events.
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

template <class T>
ens_status launch_rodas4(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return with_ode_model(model, [&](auto mt) -> ens_status {
    using M = decltype(mt);
    if constexpr (HasEvent<M>::value) return ENS_E_UNSUPPORTED;                  // events: Tsit5 only (R18)
    else if constexpr (M::n > 8 && sizeof(T) == 4) return ENS_E_UNSUPPORTED;     // POLLU: fp64 only
    else return run_rodas4<M, T>(a, opt, s);
  });
}

template ens_status launch_rodas4<float>(int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_rodas4<double>(int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
