// inputs.cuh — on-device twin of synth/inputs.py: SplitMix64 on a
// (seed, global index, slot) counter → exact uniform → p in fp64 → cast to T.
// Each rank of a sharded run generates only its own shard (no scatter, unlike
// the paper's MPI demo P:395).
#pragma once
#include "common.cuh"

namespace ens {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ double input_uniform(uint64_t seed, uint64_t g, int j) {
  const uint64_t h = mix64(seed + (g * 8ull + (uint64_t)(j + 1)) * 0x9E3779B97F4A7C15ull);
  return ((double)(h >> 12) + 0.5) * 2.220446049250313080847263336181640625e-16;
}

struct InputSpec {
  int n, m, recipe;
  double pbar[32], ubar[32];
  double n_total;
  double lo[8], hi[8];   // grid recipe ranges
  int64_t levels;        // grid recipe levels per parameter
};

template <class T>
__global__ void generate_inputs_kernel(InputSpec s, uint64_t seed, int64_t N, int64_t off, int64_t clen,
                                       int64_t cstride, T* __restrict__ u0, T* __restrict__ p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int64_t g = clen > 0 ? off + (i / clen) * cstride + i % clen : off + i;
  for (int c = 0; c < s.n; ++c) u0[(size_t)c * N + i] = (T)s.ubar[c];
  if (s.recipe == 0) {          // random10
    for (int j = 0; j < s.m; ++j) {
      const double U = input_uniform(seed, (uint64_t)g, j);
      p[(size_t)j * N + i] = (T)(s.pbar[j] * (1.0 + 0.1 * (2.0 * U - 1.0)));
    }
  } else if (s.recipe == 1) {   // rho_sweep (Lorenz)
    p[i] = (T)10.0;
    p[(size_t)N + i] = (T)((21.0 * (double)(g + 1)) / s.n_total);
    p[(size_t)2 * N + i] = (T)(8.0 / 3.0);
  } else if (s.recipe == 3) {   // grid (CRN): digit j of g in base L, parameter j fastest-first
    int64_t r = g;
    double nu0 = 0.0;
    for (int j = 0; j < s.m; ++j) {
      const int64_t d = r % s.levels;
      r /= s.levels;
      const double v = (s.hi[j] - s.lo[j]) * ((double)d / (double)(s.levels - 1)) + s.lo[j];
      p[(size_t)j * N + i] = (T)v;
      if (j == 3) nu0 = v;
    }
    for (int c = 0; c < s.n; ++c) u0[(size_t)c * N + i] = (T)nu0;   // u0 = ν0
  } else if (i == 0) {          // const: p̄ broadcast
    for (int j = 0; j < s.m; ++j) p[j] = (T)s.pbar[j];
  }
}

}  // namespace ens
