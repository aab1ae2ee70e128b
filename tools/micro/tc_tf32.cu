// tcgen05.mma kind::tf32 on sm_100a: checks the operand layout / descriptor encoding used
// by the sorted-mode tensor-core evaluation (cudagen.py, tc=1) and measures its rate.
//
//   D[128 x N] = A[128 x K] . B[N x K]^T   (both operands K-major, no swizzle, f32 accumulate)
//
// smem layout of an R x K operand (the canonical "interleaved" K-major UMMA layout):
//   element (r, k) at  (k / 4) * (R * 16) + r * 16 + (k % 4) * 4  bytes
// i.e. core matrices of 8 rows x 16 B; SBO (8-row group stride) = 128 B, LBO (stride of the
// two 16-B K chunks of one K=8 MMA step) = R * 16 B.
//
// Test 1: plain TF32 product vs fp64 (expect ~1e-3 relative: 10-bit mantissas).
// Test 2: 3-pass split (A_hi B_hi + A_hi B_lo + A_lo B_hi, hi = tf32 truncation) vs fp64
//         (expect ~1e-6: the error-compensated form the evaluation uses).
// Test 3: throughput of back-to-back MMAs (M=128, N=96, K=8 each) on every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_tf32 tc_tf32.cu && ./tc_tf32
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int M = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version 1 (sm_100)
  return d;                  // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D f32
       | (2u << 7)            // A tf32
       | (2u << 10)           // B tf32
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(cnt) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {   // truncate to the 10 mantissa bits tf32 keeps
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// one CTA of 128 threads: thread r owns row r of A and (r < N) row r of B
template <int N, int K>
__global__ void __launch_bounds__(128) tc_test(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* a_hi = reinterpret_cast<float*>(sm);
  float* a_lo = a_hi + M * K;
  float* b_hi = a_lo + M * K;
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int r = threadIdx.x, w = r >> 5;
  for (int k = 0; k < K; ++k) {
    const float v = A[r * K + k];
    const float h = split ? tf32_hi(v) : v;
    a_hi[(k / 4) * (M * 4) + r * 4 + (k % 4)] = h;
    a_lo[(k / 4) * (M * 4) + r * 4 + (k % 4)] = v - h;
    if (r < N) {
      const float bv = B[r * K + k];
      const float bh = split ? tf32_hi(bv) : bv;
      b_hi[(k / 4) * (N * 4) + r * 4 + (k % 4)] = bh;
      b_lo[(k / 4) * (N * 4) + r * 4 + (k % 4)] = bv - bh;
    }
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (r == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // st.shared -> async proxy
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (r == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t aoff = s * 2 * M * 16, boff = s * 2 * N * 16;
      mma_tf32(tm, sdesc(smem_u32(a_hi) + aoff, M * 16, 128), sdesc(smem_u32(b_hi) + boff, N * 16, 128), idesc, s > 0);
      if (split) {
        mma_tf32(tm, sdesc(smem_u32(a_hi) + aoff, M * 16, 128), sdesc(smem_u32(b_lo) + boff, N * 16, 128), idesc, 1);
        mma_tf32(tm, sdesc(smem_u32(a_lo) + aoff, M * 16, 128), sdesc(smem_u32(b_hi) + boff, N * 16, 128), idesc, 1);
      }
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(32 * w) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[r * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tm));
}

// throughput: every CTA issues `iters` x (K/8) MMAs into its own TMEM accumulator
template <int N, int K>
__global__ void __launch_bounds__(128) tc_rate(int iters, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* a = reinterpret_cast<float*>(sm);
  float* b = a + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int r = threadIdx.x, w = r >> 5;
  for (int i = r; i < (M + N) * K; i += 128) a[i] = 1.0f / (1 + (i & 7));
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (r == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (r == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int it = 0; it < iters; ++it)
      for (int s = 0; s < K / 8; ++s)
        mma_tf32(tm, sdesc(smem_u32(a) + s * 2 * M * 16, M * 16, 128),
                 sdesc(smem_u32(b) + s * 2 * N * 16, N * 16, 128), idesc, it + s > 0);
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (r == 0) sink[blockIdx.x] = __uint_as_float(v);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tm));
}

// A operand from TMEM (tcgen05.st of each thread's row), B from smem
__device__ __forceinline__ void mma_tf32_ts(uint32_t dtmem, uint32_t atmem, uint64_t bd, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
               :: "r"(dtmem), "r"(atmem), "l"(bd), "r"(idesc), "r"(acc));
}

template <int N, int K>
__global__ void __launch_bounds__(128) tc_test_ts(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* b_hi = reinterpret_cast<float*>(sm);
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int r = threadIdx.x, w = r >> 5;
  for (int k = 0; k < K; ++k) {
    if (r < N) {
      const float bv = B[r * K + k];
      const float bh = split ? tf32_hi(bv) : bv;
      b_hi[(k / 4) * (N * 4) + r * 4 + (k % 4)] = bh;
      b_lo[(k / 4) * (N * 4) + r * 4 + (k % 4)] = bv - bh;
    }
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (r == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t a_hi = tm + 128, a_lo = tm + 128 + K;   // columns after D
  // each thread writes its row of A (hi, lo) into TMEM lane r
  for (int k0 = 0; k0 < K; k0 += 8) {
    uint32_t h[8], l[8];
    for (int j = 0; j < 8; ++j) {
      const float v = A[r * K + k0 + j];
      const float hv = split ? tf32_hi(v) : v;
      h[j] = __float_as_uint(hv);
      l[j] = __float_as_uint(v - hv);
    }
    const uint32_t lane = (uint32_t)(32 * w) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(a_hi + lane + k0), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(a_lo + lane + k0), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (r == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t boff = s * 2 * N * 16;
      mma_tf32_ts(tm, a_hi + s * 8, sdesc(smem_u32(b_hi) + boff, N * 16, 128), idesc, s > 0);
      if (split) {
        mma_tf32_ts(tm, a_hi + s * 8, sdesc(smem_u32(b_lo) + boff, N * 16, 128), idesc, 1);
        mma_tf32_ts(tm, a_lo + s * 8, sdesc(smem_u32(b_hi) + boff, N * 16, 128), idesc, 1);
      }
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(32 * w) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[r * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
}

int main() {
  constexpr int N = 96, K = 24;
  float *hA = new float[M * K], *hB = new float[N * K], *hD = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (float)rand() / RAND_MAX;
  for (int i = 0; i < N * K; ++i) hB[i] = ((float)rand() / RAND_MAX - 0.5f) * 37.0f / 216.0f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, M * K * 4));
  CK(cudaMalloc(&dB, N * K * 4));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB, N * K * 4, cudaMemcpyHostToDevice));
  const int smem = (2 * M * K + 2 * N * K) * 4;
  CK(cudaFuncSetAttribute(tc_test<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int ok = 1;
  CK(cudaFuncSetAttribute(tc_test_ts<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * N * K * 4));
  for (int variant = 0; variant < 4; ++variant) {
    const int split = variant & 1, ts = variant >> 1;
    if (ts) tc_test_ts<N, K><<<1, 128, 2 * N * K * 4>>>(dA, dB, dD, split);
    else tc_test<N, K><<<1, 128, smem>>>(dA, dB, dD, split);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxabs = 0, scale = 0;
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < K; ++k) { ref += (double)hA[r * K + k] * hB[n * K + k]; mag += fabs((double)hA[r * K + k] * hB[n * K + k]); }
        const double e = fabs(hD[r * N + n] - ref);
        maxabs = fmax(maxabs, e);
        maxrel = fmax(maxrel, e / fmax(mag, 1e-30));
        scale = fmax(scale, mag);
      }
    printf("{\"a_operand\": \"%s\", \"test\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"max_abs_err\": %.3e, \"max_err_rel_to_sum_abs\": %.3e}\n",
           ts ? "tmem" : "smem", split ? "tf32x3_split" : "tf32_plain", M, N, K, maxabs, maxrel);
    if (split && maxrel > 1e-5) ok = 0;
    if (!split && maxrel > 5e-3) ok = 0;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rsm = (M + N) * K * 4;
  CK(cudaFuncSetAttribute(tc_rate<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, rsm));
  float* sink;
  CK(cudaMalloc(&sink, 4096 * 4));
  for (int ctas_per_sm : {1, 2, 4}) {
    const int iters = 20000;
    tc_rate<N, K><<<sms * ctas_per_sm, 128, rsm>>>(10, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tc_rate<N, K><<<sms * ctas_per_sm, 128, rsm>>>(iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * M * N * K * (double)iters * sms * ctas_per_sm;
    printf("{\"test\": \"rate\", \"ctas_per_sm\": %d, \"M\": %d, \"N\": %d, \"K_per_mma\": 8, \"tflops_tf32\": %.1f}\n",
           ctas_per_sm, M, N, flops / ms / 1e9);
  }
  printf("{\"ok\": %s}\n", ok ? "true" : "false");
  return ok ? 0 : 1;
}
