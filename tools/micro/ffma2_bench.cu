// Microbenchmark: issue / pipe rates of FFMA (3-register), FFMA (immediate), FFMA2 (packed f32x2)
// on sm_100a.  Each thread runs 8 independent chains x ITERS iterations.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma_reg(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma_imm(float* out) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], 0.999f, 0.0001f);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  unsigned long long A = f2u(make_float2(a, a)), B = f2u(make_float2(b, b));
  for (int i = 0; i < 8; ++i) x[i] = f2u(make_float2(threadIdx.x * 0.001f + i, i * 0.5f));
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  float* out; cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    double fma_total = (double)blocks * threads * ITERS * 8;
    cudaEventRecord(e0); k_ffma_reg<<<blocks, threads>>>(out, 0.999f, 0.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA reg : %.3f ms  %.1f TFLOP/s  %.1f FMA/clk/SM\n", ms, 2 * fma_total / ms / 1e9, fma_total / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); k_ffma_imm<<<blocks, threads>>>(out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA imm : %.3f ms  %.1f TFLOP/s  %.1f FMA/clk/SM\n", ms, 2 * fma_total / ms / 1e9, fma_total / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(out, 0.999f, 0.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2    : %.3f ms  %.1f TFLOP/s  %.1f FMA/clk/SM (x2 lanes)\n", ms, 4 * fma_total / ms / 1e9, 2 * fma_total / (ms * 1e-3) / sms / (clk * 1e3));
  }
  printf("clock %d kHz, %d SMs\n", clk, sms);
  return 0;
}
