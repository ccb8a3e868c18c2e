// k_rodas4_pollu.cu — rodas4 instances for POLLU (n = 20, fp64), split from k_rodas4.cu
// so the two build in parallel (rodas4_launch.cuh).
#include "rodas4_launch.cuh"

namespace ens {

ens_status run_rodas4_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s) {
  return run_rodas4<Pollu, double>(a, opt, s);
}

}  // namespace ens
