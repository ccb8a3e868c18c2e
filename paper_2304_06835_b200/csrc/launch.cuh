// launch.cuh — launch configuration shared by the per-algorithm translation
// units (k_tsit5.cu, k_vern7.cu, k_vern9.cu, k_ros23.cu, k_rodas4.cu, k_rodas5.cu, k_rodas5p.cu, k_sde.cu,
// and the POLLU units k_ros23_pollu.cu, k_rodas4_pollu.cu, k_rodas5_pollu.cu, k_rodas5p_pollu.cu) and the
// ABI (api.cu).
// Each algorithm's kernel instances live in their own .cu so the library
// builds in parallel; api.cu only sees the launch_* entry points below.
#pragma once
#include <algorithm>
#include <cstdint>

#include "../../include/ens.h"
#include "common.cuh"
#include "models.cuh"
#include "models_stiff.cuh"
#include "sched.cuh"

namespace ens {

constexpr int kBlock = 256;

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count();   // api.cu (cached device attribute)

// Block size of a one-thread-per-trajectory launch: 256 once the ensemble
// fills every SM with 256-thread blocks, otherwise smaller (down to one warp)
// so that small ensembles — C1's 1024 trajectories, the stiff suite's 8192 —
// spread over all SMs instead of a handful (the latency-bound regime).
inline int solver_block(int64_t threads) {
  const int64_t per_sm = cdiv(threads, sm_count());
  return (int)std::min<int64_t>(kBlock, std::max<int64_t>(32, cdiv(per_sm, 32) * 32));
}
inline dim3 grid_for(int64_t N) { return dim3((unsigned)cdiv(N, solver_block(N))); }

// Register-heavy kernels (fp64 Vern9 / Rodas5 / Vern7: 120–140 registers) fit
// only one or two 256-thread blocks per SM; smaller blocks pack more warps into
// the same register file. Starting from solver_block(N), pick the block size
// (256 / 128 / 64) with the most resident warps per SM (ties: the larger).
// Results do not depend on it (one trajectory per thread).
int cached_block(const void* kernel, int b0);          // api.cu: 0 if not cached yet
void cache_block(const void* kernel, int b0, int b);    // api.cu

template <class K>
int occupancy_block(K kernel, int64_t N) {
  const int b0 = solver_block(N);
  if (const int c = cached_block((const void*)kernel, b0)) return c;
  int best_b = b0, best_w = -1;
  for (int b = b0; b >= 64; b /= 2) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, b, 0) != cudaSuccess) break;
    const int w = occ * (b / 32);
    if (w > best_w) { best_w = w; best_b = b; }
    if (b == b0 && occ * b >= 2048) break;   // already full residency
  }
  cache_block((const void*)kernel, b0, best_b);
  return best_b;
}

inline ens_status launch_status() { return cudaPeekAtLastError() == cudaSuccess ? ENS_OK : ENS_E_CUDA; }

// Adaptive solve of one lane type: static mapping (one trajectory per thread)
// or the a8 refill scheduler with a grid of exactly the resident warps.
template <class Lane, class T, int MINB = 1>
void launch_adaptive(const Args<T>& a, bool refill, cudaStream_t s) {
  if (refill) {
    auto kern = adaptive_refill_kernel<Lane, T, MINB>;
    const dim3 b(occupancy_block(kern, a.N));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (int)b.x, 0);
    const dim3 gr((unsigned)std::min<int64_t>(cdiv(a.N, b.x), (int64_t)std::max(1, occ) * sm_count()));
    kern<<<gr, b, 0, s>>>(a);
  } else {
    auto kern = adaptive_static_kernel<Lane, T, MINB>;
    const dim3 b(occupancy_block(kern, a.N));
    kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
  }
}

// One-thread-per-trajectory launch of a fixed-step kernel with the occupancy-tuned block.
template <class K, class T>
void launch_fixed(K kern, const Args<T>& a, cudaStream_t s) {
  const dim3 b(occupancy_block(kern, a.N));
  kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
}

// ODE model dispatch: calls f(M{}) with the model type for `model`.
template <class F>
ens_status with_ode_model(int model, F&& f) {
  switch (model) {
    case ENS_LORENZ: return f(Lorenz{});
    case ENS_ROBERTSON: return f(Robertson{});
    case ENS_EXPDECAY: return f(ExpDecay{});
    case ENS_HARMONIC: return f(Harmonic{});
    case ENS_OREGO: return f(Orego{});
    case ENS_HIRES: return f(Hires{});
    case ENS_POLLU: return f(Pollu{});
    case ENS_BALL: return f(Ball{});
  }
  return ENS_E_INVALID_ARG;
}

template <class T> ens_status launch_tsit5(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_ros23(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_rodas4(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_vern7(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_rodas5(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_rodas5p(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_vern9(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s);
template <class T> ens_status launch_sde(int model, int alg, const Args<T>& a, const ens_options* opt, cudaStream_t s);

}  // namespace ens
