// k_tsit5.cu — Tsit5 kernel instances (fixed step: f2-packed fp32 / fp64;
// adaptive: static or refill scheduling) for every ODE model with n ≤ 8.
#include <type_traits>

#include "launch.cuh"
#include "tsit5.cuh"

// A/B builds only (tools/build_variant.py -DENS_NO_PAIR_ADAPTIVE=1): the scalar fp32 adaptive kernel
#ifndef ENS_NO_PAIR_ADAPTIVE
#define ENS_NO_PAIR_ADAPTIVE 0
#endif

namespace ens {

// Bulk save rows must start on 16-byte boundaries: u_out aligned and ld·sizeof(T)
// a multiple of 16 (block starts are multiples of 128 B). Off by default: on the
// saveat-dense config the two block barriers per save cost more than the per-thread
// 8-byte stores they replace (15.9 vs 15.2 ms, profiles/bulk_saves_vs_stg_r01.jsonl);
// ens_options.bulk_saves = 1 selects it (tests/test_gpu_saves.py).
template <class T>
bool bulk_saves_ok(const Args<T>& a, const ens_options* opt) {
  return opt->bulk_saves == 1 && (reinterpret_cast<uintptr_t>(a.u_out) % 16) == 0 &&
         ((size_t)a.ldo * sizeof(T)) % 16 == 0;
}

template <class M, class T>
ens_status run_tsit5(const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  const bool save = a.k > 0;
  if (!opt->adaptive) {
    if constexpr (std::is_same<T, float>::value) {
      // fp32: two trajectories per thread on the packed FFMA2 path
      const auto cf = make_tsit_coef<float, float2>(a.dt0, a.h_last);
      const int64_t threads = cdiv(a.N, 2);
      if (save) {
        // the saving instances hold more registers: pick the block size with the most resident warps
        auto kern = !a.save_grid_only ? tsit5_fixed_kernel<M, f2, 1>
                    : bulk_saves_ok(a, opt) ? tsit5_fixed_kernel<M, f2, 3> : tsit5_fixed_kernel<M, f2, 2>;
        const dim3 b2(occupancy_block(kern, threads));
        const size_t smem = (a.save_grid_only && bulk_saves_ok(a, opt)) ? 2 * M::n * b2.x * 2 * sizeof(float) : 0;
        kern<<<dim3((unsigned)cdiv(threads, b2.x)), b2, smem, s>>>(a, cf);
      } else {
        // up to a few waves, the block size with the most resident warps balances the SMs better
        // (56 registers: 36 warps in 128-thread blocks vs 32 in 256; N = 10^5: 0.45 -> 0.36 ms);
        // for many waves 256-thread blocks measured 1.4 % faster (profiles/fixed_block_size_r01.jsonl)
        auto kern = opt->want_stats ? tsit5_fixed_kernel<M, f2, 0, true> : tsit5_fixed_kernel<M, f2, 0>;
        const bool few_waves = threads < (int64_t)4 * sm_count() * 1024;
        const dim3 b2(few_waves ? occupancy_block(kern, threads) : solver_block(threads));
        kern<<<dim3((unsigned)cdiv(threads, b2.x)), b2, 0, s>>>(a, cf);
      }
    } else {
      const auto cf = make_tsit_coef<double, double>(a.dt0, a.h_last);
      if (save) {
        auto kern = !a.save_grid_only ? tsit5_fixed_kernel<M, double, 1>
                    : bulk_saves_ok(a, opt) ? tsit5_fixed_kernel<M, double, 3> : tsit5_fixed_kernel<M, double, 2>;
        const dim3 b(occupancy_block(kern, a.N));
        const size_t smem = (a.save_grid_only && bulk_saves_ok(a, opt)) ? 2 * M::n * b.x * sizeof(double) : 0;
        kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, smem, s>>>(a, cf);
      } else {
        const dim3 g = grid_for(a.N), b(solver_block(a.N));
        if (opt->want_stats) tsit5_fixed_kernel<M, double, 0, true><<<g, b, 0, s>>>(a, cf);
        else tsit5_fixed_kernel<M, double, 0><<<g, b, 0, s>>>(a, cf);
      }
    }
  } else {
    // (a two-trajectories-per-thread f2 variant — packed stage / error / controller arithmetic,
    //  branch-free per-lane control — issued 194 instead of 281 thread-instructions per attempt,
    //  but at 94 registers (20 warps per SM) it is latency-bound with the FMA pipe as busy as
    //  now (66 %): 4.04 ms vs 4.09 ms, 3.98 ms capped at 80 registers; not adopted)
    // static mapping without events: the written-out loop kernel (fp64 C1-style ensembles
    // 4.31 -> 4.10 ms, fp32 C2 adaptive 4.09 -> 4.05 ms; profiles/ab_r02/)
    if constexpr (!HasEvent<M>::value) {
      if (!opt->refill) {
        if constexpr (std::is_same<T, float>::value && M::n >= 2 && !ENS_NO_PAIR_ADAPTIVE) {
          // fp32: component pairs on the packed FFMA2 path (bit-identical to the scalar kernel)
          auto kern = save ? tsit5_static_pair_kernel<M, true> : tsit5_static_pair_kernel<M, false>;
          const dim3 b(occupancy_block(kern, a.N));
          kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
          return launch_status();
        }
        auto kern = save ? tsit5_static_kernel<M, T, true> : tsit5_static_kernel<M, T, false>;
        const dim3 b(occupancy_block(kern, a.N));
        kern<<<dim3((unsigned)cdiv(a.N, b.x)), b, 0, s>>>(a);
        return launch_status();
      }
    }
    if (save) launch_adaptive<Tsit5Lane<M, T, true>, T>(a, opt->refill, s);
    else launch_adaptive<Tsit5Lane<M, T, false>, T>(a, opt->refill, s);
  }
  return launch_status();
}

template <class T>
ens_status launch_tsit5(int model, const Args<T>& a, const ens_options* opt, cudaStream_t s) {
  return with_ode_model(model, [&](auto mt) -> ens_status {
    using M = decltype(mt);
    // register-resident Tsit5 stages are instantiated for n ≤ 8 (POLLU, n = 20, is stiff-only)
    if constexpr (M::n > 8) return ENS_E_UNSUPPORTED;
    else return run_tsit5<M, T>(a, opt, s);
  });
}

template ens_status launch_tsit5<float>(int, const Args<float>&, const ens_options*, cudaStream_t);
template ens_status launch_tsit5<double>(int, const Args<double>&, const ens_options*, cudaStream_t);

}  // namespace ens
