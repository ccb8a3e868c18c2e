// k_rodas5p_pollu.cu — rodas5p instances for POLLU (n = 20, fp64), split from k_rodas5p.cu
// so the two build in parallel (rodas5_launch.cuh).
#include "rodas5_launch.cuh"

namespace ens {

ens_status run_rodas5p_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s) {
  return run_rodas5p<Pollu, double>(a, opt, s);
}

}  // namespace ens
