// k_ros23_pollu.cu — ros23 instances for POLLU (n = 20, fp64), split from k_ros23.cu
// so the two build in parallel (ros23_launch.cuh).
#include "ros23_launch.cuh"

namespace ens {

ens_status run_ros23_pollu(const Args<double>& a, const ens_options* opt, cudaStream_t s) {
  return run_ros23<Pollu, double>(a, opt, s);
}

}  // namespace ens
