// Peak-issue microbenchmarks for the roofline denominators.
// Measurement infrastructure only: not part of the solver path.
//
// Each kernel runs a register-resident loop of one instruction class over 8
// independent chains per thread on a full grid (148 SMs x 8 blocks x 256 thr),
// timed with CUDA events; FLOP/s = lanes x ops x flop_per_op / time.
// The SM clock is read with clock64() vs globaltimer inside one block so the
// per-SM-per-clock rate can be derived independently of DVFS.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// 3-register FFMA: a = a*b + c with b, c in registers.
__global__ void k_ffma_reg(float* out, float b, float c, unsigned long long* clk) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint64_t c0 = clock64(), g0 = gtimer();
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    a0 = __fmaf_rn(a0, b, c); a1 = __fmaf_rn(a1, b, c); a2 = __fmaf_rn(a2, b, c); a3 = __fmaf_rn(a3, b, c);
    a4 = __fmaf_rn(a4, b, c); a5 = __fmaf_rn(a5, b, c); a6 = __fmaf_rn(a6, b, c); a7 = __fmaf_rn(a7, b, c);
  }
  uint64_t c1 = clock64(), g1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// FFMA with an immediate multiplier (the tableau-coefficient form).
__global__ void k_ffma_imm(float* out, float c, unsigned long long* clk) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint64_t c0 = clock64(), g0 = gtimer();
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    a0 = __fmaf_rn(a0, 0.999f, c); a1 = __fmaf_rn(a1, 0.999f, c); a2 = __fmaf_rn(a2, 0.999f, c); a3 = __fmaf_rn(a3, 0.999f, c);
    a4 = __fmaf_rn(a4, 0.999f, c); a5 = __fmaf_rn(a5, 0.999f, c); a6 = __fmaf_rn(a6, 0.999f, c); a7 = __fmaf_rn(a7, 0.999f, c);
  }
  uint64_t c1 = clock64(), g1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// Packed FFMA2 (sm_100): two fp32 FMAs per lane per instruction.
__global__ void k_ffma2(float* out, float b, float c, unsigned long long* clk) {
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  float2 a0 = make_float2(threadIdx.x, 1), a1 = make_float2(2, 3), a2 = make_float2(4, 5), a3 = make_float2(6, 7);
  float2 a4 = make_float2(8, 9), a5 = make_float2(10, 11), a6 = make_float2(12, 13), a7 = make_float2(14, 15);
  uint64_t c0 = clock64(), g0 = gtimer();
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    a0 = __ffma2_rn(a0, bb, cc); a1 = __ffma2_rn(a1, bb, cc); a2 = __ffma2_rn(a2, bb, cc); a3 = __ffma2_rn(a3, bb, cc);
    a4 = __ffma2_rn(a4, bb, cc); a5 = __ffma2_rn(a5, bb, cc); a6 = __ffma2_rn(a6, bb, cc); a7 = __ffma2_rn(a7, bb, cc);
  }
  uint64_t c1 = clock64(), g1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0.x + a1.x + a2.x + a3.x + a4.y + a5.y + a6.y + a7.y;
}

// FP64 DFMA.
__global__ void k_dfma(double* out, double b, double c, unsigned long long* clk) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint64_t c0 = clock64(), g0 = gtimer();
  #pragma unroll 16
  for (int i = 0; i < ITERS / 4; ++i) {
    a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
    a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
  }
  uint64_t c1 = clock64(), g1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// Integer multiply-hi (Philox's core op).
__global__ void k_imad_hi(unsigned* out, unsigned b, unsigned long long* clk) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  uint64_t c0 = clock64(), g0 = gtimer();
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    a0 = __umulhi(a0, b) ^ a1; a1 = __umulhi(a1, b) ^ a2; a2 = __umulhi(a2, b) ^ a3; a3 = __umulhi(a3, b) ^ a0;
    a4 = __umulhi(a4, b) ^ a5; a5 = __umulhi(a5, b) ^ a6; a6 = __umulhi(a6, b) ^ a7; a7 = __umulhi(a7, b) ^ a4;
  }
  uint64_t c1 = clock64(), g1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"attr_clock_mhz\": %.0f, \"regs_per_sm\": %d}\n",
         prop.name, sms, prop.major, prop.minor, clk_khz / 1e3, prop.regsPerMultiprocessor);
  const int threads = 256, blocks = sms * 8;
  const size_t nthr = (size_t)threads * blocks;
  float* fo; double* dout; unsigned* uo; unsigned long long* clk;
  CK(cudaMalloc(&fo, nthr * 4)); CK(cudaMalloc(&dout, nthr * 8)); CK(cudaMalloc(&uo, nthr * 4));
  CK(cudaMalloc(&clk, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct R { const char* name; double ops_per_thread; double flop_per_op; };
  for (int which = 0; which < 5; ++which) {
    double best_ms = 1e30; unsigned long long hc[2] = {0, 0};
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      switch (which) {
        case 0: k_ffma_reg<<<blocks, threads>>>(fo, 0.999f, 1e-3f, clk); break;
        case 1: k_ffma_imm<<<blocks, threads>>>(fo, 1e-3f, clk); break;
        case 2: k_ffma2<<<blocks, threads>>>(fo, 0.999f, 1e-3f, clk); break;
        case 3: k_dfma<<<blocks, threads>>>(dout, 0.999, 1e-3, clk); break;
        case 4: k_imad_hi<<<blocks, threads>>>(uo, 0xD2511F53u, clk); break;
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best_ms) { best_ms = ms; CK(cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost)); }
    }
    const char* names[] = {"ffma_reg", "ffma_imm", "ffma2", "dfma", "imad_hi"};
    double ops = (which == 3 ? ITERS / 4 : ITERS) * 8.0 * nthr;         // warp-lane instructions
    double flop_per = (which == 2 ? 4.0 : (which == 4 ? 1.0 : 2.0));    // per lane-instruction
    double rate = ops * flop_per / (best_ms * 1e-3);
    double sm_mhz = hc[1] ? (double)hc[0] / (double)hc[1] * 1e3 : 0.0;
    // per-SM per-clock lane-ops (the hardware rate independent of DVFS)
    double per_sm_clk = ops / (best_ms * 1e-3) / sms / (sm_mhz * 1e6);
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"rate_per_s\": %.4e, \"unit\": \"%s\", \"sm_mhz_measured\": %.0f, "
           "\"lane_instr_per_sm_per_clk\": %.2f}\n",
           names[which], best_ms, rate, which == 4 ? "imad_hi/s" : "FLOP/s", sm_mhz, per_sm_clk);
  }
  return 0;
}
