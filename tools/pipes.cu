// Does scalar FFMA (fmalite) co-issue with packed FFMA2 (fmaheavy)? Measures
// FMA/SM/clk for: pure FFMA, pure FFMA2, and interleaved mixes.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 2048;
template <int MIX>   // per iteration: 8 FFMA2 chains + MIX scalar FFMA chains
__global__ void k(float* out, float b, float c, unsigned long long* clk) {
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  float2 a[8]; float s[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x + i, i); s[i] = threadIdx.x * 0.5f + i; }
  long long c0 = clock64();
#pragma unroll 4
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], bb, cc);
#pragma unroll
    for (int i = 0; i < MIX; ++i) s[i] = __fmaf_rn(s[i], b, c);
  }
  long long c1 = clock64();
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y + s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = c1 - c0;
}
__global__ void kscalar(float* out, float b, float c, unsigned long long* clk) {
  float s[16]; for (int i = 0; i < 16; ++i) s[i] = threadIdx.x + i;
  long long c0 = clock64();
#pragma unroll 4
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = __fmaf_rn(s[i], b, c);
  long long c1 = clock64();
  float r = 0; for (int i = 0; i < 16; ++i) r += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = c1 - c0;
}
template <class F> void run(const char* name, F f, double fma_per_thread_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  float* o; unsigned long long* clk; cudaMalloc(&o, blocks * threads * 4); cudaMalloc(&clk, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f; unsigned long long cy = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(blocks, threads, o, clk); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) { best = ms; cudaMemcpy(&cy, clk, 8, cudaMemcpyDeviceToHost); }
  }
  const double fmas = (double)blocks * threads * IT * fma_per_thread_iter;
  const double mhz = 1965.0;
  printf("{\"case\": \"%s\", \"ms\": %.4f, \"fma_per_sm_per_clk_at_1965\": %.1f, \"TFLOPs\": %.2f}\n", name, best,
         fmas / (best * 1e-3) / sms / (mhz * 1e6), 2 * fmas / (best * 1e-3) / 1e12);
}
int main() {
  run("ffma scalar x16", [](int b, int t, float* o, unsigned long long* c) { kscalar<<<b, t>>>(o, 0.999f, 1e-3f, c); }, 16);
  run("ffma2 x8", [](int b, int t, float* o, unsigned long long* c) { k<0><<<b, t>>>(o, 0.999f, 1e-3f, c); }, 16);
  run("ffma2 x8 + ffma x4", [](int b, int t, float* o, unsigned long long* c) { k<4><<<b, t>>>(o, 0.999f, 1e-3f, c); }, 20);
  run("ffma2 x8 + ffma x8", [](int b, int t, float* o, unsigned long long* c) { k<8><<<b, t>>>(o, 0.999f, 1e-3f, c); }, 24);
  return 0;
}
