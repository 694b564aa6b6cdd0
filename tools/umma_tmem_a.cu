// Probe: tcgen05.mma kind::tf32 with the A operand in tensor memory (lane = row m, one tf32 per
// 32-bit column along K) and B in shared memory (K-major, no swizzle). Checks D = A·B^T against a
// host reference (1xTF32 inputs, so the comparison is exact up to fp32 accumulation order), then
// times chains of MMAs per SM for several N, next to the same chain with A in shared memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_tmem_a tools/umma_tmem_a.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ inline uint32_t kmaj(int row, int k, int rows) {
  return (uint32_t)((k >> 2) * (rows / 8) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (uint64_t)((lbo >> 4) & 0x3FFF) << 16 |
         (uint64_t)((sbo >> 4) & 0x3FFF) << 32 | (uint64_t)1 << 46;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void wait_bar(uint64_t* b, int parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity));
}

constexpr int K = 16;  // two MMAs of K = 8
constexpr int ACOL = 256;  // TMEM column of A

// mode 0: A from TMEM, mode 1: A from smem. iters chains of 2 MMAs; D written to out when iters == 1.
__global__ void run(const float* A, const float* B, float* out, int n, int iters, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* a_s = sm;              // [128][K] K-major
  unsigned char* b_s = sm + 128 * K * 4;  // [n][K]
  for (int i = tid; i < 128 * K; i += blockDim.x)
    *reinterpret_cast<float*>(a_s + kmaj(i / K, i % K, 128)) = A[i];
  for (int i = tid; i < n * K; i += blockDim.x) *reinterpret_cast<float*>(b_s + kmaj(i / K, i % K, n)) = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  {  // A into TMEM: warp w writes lanes 32w..32w+31, K columns from ACOL
    const int row = 32 * warp + lane;
    uint32_t v[K];
    for (int k = 0; k < K; ++k) v[k] = __float_as_uint(A[row * K + k]);
    const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + ACOL;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, n), lboA = 16 * 128, lboB = (n / 8) * 128;
    const uint32_t b0 = smem_u32(b_s), a0 = smem_u32(a_s);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t bd = smem_desc(b0 + ks * 2 * lboB, lboB, 128);
        const uint32_t acc = (it | ks) ? 1u : 0u;
        if (mode == 0) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + ACOL + ks * 8), "l"(bd), "r"(idesc), "r"(acc));
        } else {
          const uint64_t ad = smem_desc(a0 + ks * 2 * lboA, lboA, 128);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  wait_bar(&mbar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (iters == 1 && blockIdx.x == 0)
    for (int c0 = 0; c0 < n; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) out[(32 * warp + lane) * n + c0 + j] = __uint_as_float(v[j]);
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static float tf32(float x) {  // truncate to tf32 (exact input for the MMA)
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int smem = (128 + 256) * K * 4;
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 128 * K * 4);
  cudaMalloc(&dB, 256 * K * 4);
  cudaMalloc(&dD, 128 * 256 * 4);
  std::vector<float> A(128 * K), B(256 * K), D(128 * 256);
  uint32_t seed = 12345;
  auto rnd = [&]() { seed = seed * 1664525u + 1013904223u; return tf32(((seed >> 8) / 16777216.0f) * 2.f - 1.f); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int ns[] = {48, 96, 128};
  for (int n : ns)
    for (int mode = 0; mode < 2; ++mode) {
      run<<<1, 128, smem>>>(dA, dB, dD, n, 1, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"n\": %d, \"mode\": %d, \"error\": \"%s\"}\n", n, mode, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(D.data(), dD, 128 * n * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int m = 0; m < 128; ++m)
        for (int j = 0; j < n; ++j) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[j * K + k];
          err = fmax(err, fabs(ref - D[m * n + j]));
        }
      const int iters = 20000;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      run<<<sms, 128, smem>>>(dA, dB, dD, n, iters, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"n\": %d, \"a_operand\": \"%s\", \"max_abs_err\": %.3e, \"cycles_per_mma\": %.2f}\n", n,
             mode == 0 ? "tmem" : "smem", err, ms / 1e3 * clk_khz * 1e3 / (2.0 * iters));
    }
  return 0;
}
