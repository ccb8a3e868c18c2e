// k_rodas5p.cu — Rodas5P kernel instances (R23; fixed step with grid saves;
// adaptive static or refill; dense output by shortened steps, DESIGN R24) for the ODE models without events.
#include <type_traits>

#include "rodas5_launch.cuh"

namespace ens {

template <class T>
ens_status launch_rodas5p(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return with_ode_model(model, [&](auto mt) -> ens_status {
    using M = decltype(mt);
    if constexpr (HasEvent<M>::value) return ENS_E_UNSUPPORTED;                  // events: Tsit5 only (R18)
    else if constexpr (M::n > 8 && sizeof(T) == 4) return ENS_E_UNSUPPORTED;     // POLLU: fp64 only
    else if constexpr (std::is_same<M, Pollu>::value) return run_rodas5p_pollu(a, opt, s);   // k_rodas5p_pollu.cu
    else return run_rodas5p<M, T>(a, opt, s);
  });
}

template ens_status launch_rodas5p<float>(int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_rodas5p<double>(int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
