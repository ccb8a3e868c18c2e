// k_vern9.cu — Vern9 kernel instances (fixed step; adaptive static or refill)
// for the non-stiff ODE models with n ≤ 8 and no events (DESIGN R21).
#include "verner_launch.cuh"

namespace ens {

template <class T>
ens_status launch_vern9(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return launch_verner_tab<Vern9Tab, T>(model, a, opt, s);
}

template ens_status launch_vern9<float>(int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_vern9<double>(int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
