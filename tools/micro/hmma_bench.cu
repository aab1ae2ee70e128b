// Legacy warp-level MMA (mma.sync -> HMMA) throughput on sm_100a: TF32 m16n8k8 and
// BF16 m16n8k16, f32 accumulate.  Each warp keeps 8 independent accumulators in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_bench hmma_bench.cu && ./hmma_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void bench(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float acc[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[k][0]), "+f"(acc[k][1]), "+f"(acc[k][2]), "+f"(acc[k][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[k][0]), "+f"(acc[k][1]), "+f"(acc[k][2]), "+f"(acc[k][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1 << 26);
  for (int kind = 0; kind < 2; ++kind) {
    for (int wpb : {4, 8, 16}) {
      const int iters = 4096, blocks = sms * 2;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto run = [&] {
        if (kind == 0) bench<0><<<blocks, 32 * wpb>>>(out, iters);
        else bench<1><<<blocks, 32 * wpb>>>(out, iters);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops_per_mma = kind == 0 ? 16.0 * 8 * 8 * 2 : 16.0 * 8 * 16 * 2;
      const double tot = (double)blocks * wpb * iters * 8 * flops_per_mma;
      printf("%s warps/CTA %2d x %d CTAs: %.3f ms  %.1f TFLOP/s\n", kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16",
             wpb, blocks, ms, tot / ms / 1e9);
    }
  }
  return 0;
}
