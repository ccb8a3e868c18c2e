// stats.cuh — deterministic ensemble statistics ("mean and variance of
// the solution"; DESIGN R12): (count, mean, M2) over the finite values of each
// (save point, component) row, per block by two passes over the block's values,
// then merged across blocks by Chan's pairwise update in a fixed order. Never
// depends on scheduling, so a fixed N and launch give bit-identical results.
#pragma once
#include "common.cuh"

namespace ens {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in fixed order; `red` is shared scratch of >= 32 doubles.
// Must be called by every thread of the block.
__device__ __forceinline__ double block_sum(double* red, double v) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();                      // red may still be read by a previous call
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
  }
  if (threadIdx.x == 0) red[0] = r;
  __syncthreads();
  return red[0];
}

// Two-pass (count, mean, M2) of the block's finite values; thread 0 writes out3.
__device__ __forceinline__ void block_stats_partial(double* red, bool valid, double x, double* out3) {
  const bool use = valid && isfinite(x);
  const double c = block_sum(red, use ? 1.0 : 0.0);
  const double s = block_sum(red, use ? x : 0.0);
  const double mean = c > 0.0 ? s / c : 0.0;
  const double d = use ? x - mean : 0.0;
  const double m2 = block_sum(red, d * d);
  if (threadIdx.x == 0) { out3[0] = c; out3[1] = mean; out3[2] = m2; }
}

// Two-pass (count, mean, M2) of a warp's finite values, W per lane (fixed-step
// Tsit5 epilogue: fused statistics of the final states, one partial per warp);
// lane 0 writes out3. Every lane of the warp must call it.
template <int W>
__device__ __forceinline__ void warp_stats_partial(const bool (&use)[W], const double (&x)[W], double* out3) {
  double c = 0.0, s = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (use[w]) { c += 1.0; s += x[w]; }
  c = warp_sum(c);
  s = warp_sum(s);
  const double mean = c > 0.0 ? s / c : 0.0;
  double m2 = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (use[w]) { const double d = x[w] - mean; m2 = fma(d, d, m2); }
  m2 = warp_sum(m2);
  if ((threadIdx.x & 31) == 0) { out3[0] = c; out3[1] = mean; out3[2] = m2; }
}

struct Moments { double c, mean, m2; };

// Chan et al. pairwise combination of (count, mean, M2).
__device__ __forceinline__ Moments chan_merge(Moments a, Moments b) {
  if (b.c == 0.0) return a;
  if (a.c == 0.0) return b;
  const double c = a.c + b.c;
  const double delta = b.mean - a.mean;
  Moments r;
  r.c = c;
  r.mean = a.mean + delta * (b.c / c);
  r.m2 = a.m2 + b.m2 + delta * delta * (a.c * (b.c / c));
  return r;
}

// gridDim.y is capped at 65535: row-indexed kernels take grid.y = min(rows, kMaxGridY)
// and stride over their rows (every block of a row does the same work, so the
// block-wide barriers inside stay uniform).
constexpr int kMaxGridY = 65535;

// Partials over a stored [rows][N] array in T: grid (nparts, min(rows, 65535));
// block b reduces elements [b*chunk, (b+1)*chunk) of each of its rows.
template <class T>
__global__ void __launch_bounds__(256) stats_partial_kernel(const T* __restrict__ x, int64_t N, int64_t ld,
                                                            int64_t chunk, double* __restrict__ partial, int rows) {
  __shared__ double red[32];
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(N, lo + chunk);
  const T* xr = x + (size_t)row * ld;
  double c = 0, s = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = (double)xr[i];
    if (isfinite(v)) { c += 1.0; s += v; }
  }
  c = block_sum(red, c);
  s = block_sum(red, s);
  const double mean = c > 0 ? s / c : 0.0;
  double m2 = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = (double)xr[i];
    if (isfinite(v)) { const double d = v - mean; m2 = fma(d, d, m2); }
  }
  m2 = block_sum(red, m2);
  if (threadIdx.x == 0) {
    double* o = partial + ((size_t)row * gridDim.x + blockIdx.x) * 3;
    o[0] = c; o[1] = mean; o[2] = m2;
  }
  }
}

// Merge partials [rows][nparts][3] → out [rows][3], one 256-thread block per
// row: thread t folds parts t, t+256, … in order; then a fixed binary tree.
static __global__ void __launch_bounds__(256) stats_merge_kernel(const double* __restrict__ partial, int nparts,
                                                          double* __restrict__ out) {
  __shared__ double sc[256], sm[256], s2[256];
  const int row = blockIdx.x;
  const double* pr = partial + (size_t)row * nparts * 3;
  Moments acc{0, 0, 0};
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) acc = chan_merge(acc, Moments{pr[3 * b], pr[3 * b + 1], pr[3 * b + 2]});
  sc[threadIdx.x] = acc.c; sm[threadIdx.x] = acc.mean; s2[threadIdx.x] = acc.m2;
  __syncthreads();
  for (int w = blockDim.x >> 1; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      Moments r = chan_merge(Moments{sc[threadIdx.x], sm[threadIdx.x], s2[threadIdx.x]},
                             Moments{sc[threadIdx.x + w], sm[threadIdx.x + w], s2[threadIdx.x + w]});
      sc[threadIdx.x] = r.c; sm[threadIdx.x] = r.mean; s2[threadIdx.x] = r.m2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[row * 3] = sc[0]; out[row * 3 + 1] = sm[0]; out[row * 3 + 2] = s2[0]; }
}

// First stage of a two-stage merge for many partials (fused per-warp
// statistics: N/64 partials per row): grid (nblk, rows); block b folds partials
// [b·256·kFold, (b+1)·256·kFold) of its row — thread t folds kFold consecutive
// partials in order, then the block's fixed binary tree — into out
// [rows][nblk][3], which stats_merge_kernel then merges. Fixed order throughout.
constexpr int kFold = 8;
static __global__ void __launch_bounds__(256) stats_fold_kernel(const double* __restrict__ partial, int64_t nparts,
                                                         double* __restrict__ out, int rows) {
  __shared__ double sc[256], sm[256], s2[256];
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
  const double* pr = partial + (size_t)row * nparts * 3;
  const int64_t lo = ((int64_t)blockIdx.x * 256 + threadIdx.x) * kFold;
  Moments acc{0, 0, 0};
  for (int j = 0; j < kFold; ++j) {
    const int64_t b = lo + j;
    if (b < nparts) acc = chan_merge(acc, Moments{pr[3 * b], pr[3 * b + 1], pr[3 * b + 2]});
  }
  sc[threadIdx.x] = acc.c; sm[threadIdx.x] = acc.mean; s2[threadIdx.x] = acc.m2;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      Moments r = chan_merge(Moments{sc[threadIdx.x], sm[threadIdx.x], s2[threadIdx.x]},
                             Moments{sc[threadIdx.x + w], sm[threadIdx.x + w], s2[threadIdx.x + w]});
      sc[threadIdx.x] = r.c; sm[threadIdx.x] = r.mean; s2[threadIdx.x] = r.m2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = out + ((size_t)row * gridDim.x + blockIdx.x) * 3;
    o[0] = sc[0]; o[1] = sm[0]; o[2] = s2[0];
  }
  __syncthreads();   // the shared arrays are reused by the next row
  }
}

// Cross-rank merge: gathered [R][rows][3] folded in rank order 0..R−1.
static __global__ void stats_rank_merge_kernel(const double* __restrict__ g, int R, int rows, double* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  Moments acc{0, 0, 0};
  for (int r = 0; r < R; ++r) {
    const double* q = g + ((size_t)r * rows + row) * 3;
    acc = chan_merge(acc, Moments{q[0], q[1], q[2]});
  }
  out[row * 3] = acc.c; out[row * 3 + 1] = acc.mean; out[row * 3 + 2] = acc.m2;
}

static __global__ void stats_finalize_kernel(const double* __restrict__ st, int rows, double* __restrict__ mean,
                                      double* __restrict__ var) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const double c = st[row * 3];
  mean[row] = st[row * 3 + 1];
  var[row] = c > 1.0 ? st[row * 3 + 2] / (c - 1.0) : 0.0;
}

}  // namespace ens
