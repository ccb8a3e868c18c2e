// sched.cuh — how lanes are mapped to trajectories for adaptive solves.
//
// static: one trajectory per thread for the whole integration (Listing 1,
//   P:287-307). A warp runs until its slowest lane finishes — the thread
//   divergence the paper attributes to adaptive stepping.
// refill (a8): persistent warps; after every attempted step the warp ballots
//   its finished lanes, the leader claims that many new trajectory indices with
//   one atomicAdd on a global counter, and shuffles them to the idle lanes, so
//   finished lanes are retired and refilled instead of idling. Per-trajectory
//   arithmetic is unchanged, so results are bit-identical to `static`.
#pragma once
#include "common.cuh"

namespace ens {

// MINB: minimum resident 256-thread blocks per SM requested from ptxas (caps
// registers per thread; fp64 Rosenbrock23 runs at 3 instead of 2).
template <class Lane, class T, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) adaptive_static_kernel(const Args<T> a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  Lane L;
  L.init(a, i);
  while (!L.done) L.step(a, i);
  L.finish(a, i);
}

template <class Lane, class T, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) adaptive_refill_kernel(const Args<T> a) {
  constexpr unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  Lane L;
  L.done = true;
  int64_t idx = 0;
  bool exhausted = false;   // warp-uniform
  for (;;) {
    if (!exhausted) {
      const unsigned need = __ballot_sync(FULL, L.done);
      if (need) {
        const int cnt = __popc(need);
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if ((int)lane == leader) base = atomicAdd(a.counter, (unsigned long long)cnt);
        base = __shfl_sync(FULL, base, leader);
        if (base + (unsigned long long)cnt >= (unsigned long long)a.N) exhausted = true;
        if (L.done) {
          const int64_t cand = (int64_t)base + __popc(need & ((1u << lane) - 1u));
          if (cand < a.N) {
            idx = cand;
            L.init(a, idx);
            if (L.done) L.finish(a, idx);
          }
        }
      }
    }
    const bool active = !L.done;
    if (!__any_sync(FULL, active)) {
      if (exhausted) break;
      continue;
    }
    if (active) {
      L.step(a, idx);
      if (L.done) L.finish(a, idx);
    }
  }
}

}  // namespace ens
