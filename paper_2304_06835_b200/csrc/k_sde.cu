// k_sde.cu — Euler–Maruyama and SIEA kernel instances for the SDE models.
#include "em.cuh"
#include "launch.cuh"

namespace ens {

template <class M, class T>
ens_status run_sde(int alg, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const dim3 g = grid_for(a.N), b(solver_block(a.N));
  if (alg == ENS_SIEA) {
    if constexpr (M::nw == M::n) {   // diagonal noise only
      if (opt->want_stats) em_kernel<M, T, true, true><<<g, b, 0, s>>>(a);
      else em_kernel<M, T, false, true><<<g, b, 0, s>>>(a);
    } else {
      return ENS_E_UNSUPPORTED;
    }
  } else {
    // register caps only pay when the ensemble fills the SMs beyond two blocks each (cf. k_ros23.cu)
    const bool large = a.N > (int64_t)sm_count() * 2 * 256;
    if (!large) {
      if (opt->want_stats) em_kernel<M, T, true><<<g, b, 0, s>>>(a);
      else em_kernel<M, T, false><<<g, b, 0, s>>>(a);
    } else if constexpr (sizeof(T) == 8 && M::nw > 3) {   // fp64 CRN: three blocks per SM (em_kernel_b3)
      if (opt->want_stats) em_kernel_b3<M, T, true><<<g, b, 0, s>>>(a);
      else em_kernel_b3<M, T, false><<<g, b, 0, s>>>(a);
    } else if constexpr (sizeof(T) == 4 && M::nw == 3) {   // fp32 C4: four blocks per SM (72 -> 64 regs, 1-3 %)
      if (opt->want_stats) em_kernel_b4<M, T, true><<<g, b, 0, s>>>(a);
      else em_kernel_b4<M, T, false><<<g, b, 0, s>>>(a);
    } else {
      if (opt->want_stats) em_kernel<M, T, true><<<g, b, 0, s>>>(a);
      else em_kernel<M, T, false><<<g, b, 0, s>>>(a);
    }
  }
  return launch_status();
}

template <class T>
ens_status launch_sde(int model, int alg, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  switch (model) {
    case ENS_LORENZ_SDE_ADD: return run_sde<LorenzSDE<false>, T>(alg, a, opt, s);
    case ENS_LORENZ_SDE_MUL: return run_sde<LorenzSDE<true>, T>(alg, a, opt, s);
    case ENS_GBM: return run_sde<GBM, T>(alg, a, opt, s);
    case ENS_CRN: return run_sde<CRN, T>(alg, a, opt, s);
  }
  return ENS_E_INVALID_ARG;
}

template ens_status launch_sde<float>(int, int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_sde<double>(int, int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
