// k_vern7.cu — Vern7 kernel instances (fixed step; adaptive static or refill)
// for the non-stiff ODE models with n ≤ 8 and no events.
#include "launch.cuh"
#include "vern7.cuh"

namespace ens {

template <class M, class T>
ens_status run_vern7(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    const dim3 g = grid_for(a.N), b(solver_block(a.N));
    if (save) vern7_fixed_kernel<M, T, true><<<g, b, 0, s>>>(a);
    else vern7_fixed_kernel<M, T, false><<<g, b, 0, s>>>(a);
  } else {
    if (save) launch_adaptive<Vern7Lane<M, T, true>, T>(a, opt->refill, s);
    else launch_adaptive<Vern7Lane<M, T, false>, T>(a, opt->refill, s);
  }
  return launch_status();
}

template <class T>
ens_status launch_vern7(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return with_ode_model(model, [&](auto mt) -> ens_status {
    using M = decltype(mt);
    if constexpr (HasEvent<M>::value || M::n > 8) return ENS_E_UNSUPPORTED;   // events: Tsit5; n = 20: stiff only
    else return run_vern7<M, T>(a, opt, s);
  });
}

template ens_status launch_vern7<float>(int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_vern7<double>(int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
