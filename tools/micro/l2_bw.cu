// L2 read bandwidth on B200: all SMs stream 16-B ld.global.cg loads over an
// L2-resident buffer (default 32 MiB) many times; also an HBM-sized buffer for contrast.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ p, size_t n4, int reps, float* out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v = __ldcg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  float* out; cudaMalloc(&out, 4);
  const size_t sizes[] = {8ull << 20, 32ull << 20, 64ull << 20, 1024ull << 20};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"results\": [", sms, l2);
  for (int si = 0; si < 4; ++si) {
    size_t bytes = sizes[si];
    float4* p; cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes);
    size_t n4 = bytes / 16;
    int reps = (int)((8ull << 30) / bytes); if (reps < 2) reps = 2;
    rd<<<sms * 8, 512>>>(p, n4, 1, out);   // warm
    cudaEventRecord(a);
    rd<<<sms * 8, 512>>>(p, n4, reps, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
    printf("%s{\"buffer_mib\": %zu, \"gb_s\": %.1f}", si ? ", " : "", bytes >> 20, gbs);
    cudaFree(p);
  }
  printf("]}\n");
  return 0;
}
