// Probe for the tcgen05 (UMMA) kind::tf32 encodings used by the structured kernels:
// smem matrix descriptors (K-major, no swizzle), the instruction descriptor, TMEM alloc,
// commit/mbarrier completion and tcgen05.ld read-back. One CTA computes
//   D[M=128][N] = A[128][K] · B[N][K]^T      (tf32 inputs, fp32 accumulate)
// for 1xTF32 and 3xTF32 (hi/lo split) and prints the max relative error against fp64.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 96, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 B; element (row, k) of a [rows][K] operand at
//   (k/4) * (rows/8 * 128) + (row/8) * 128 + (row%8) * 16 + (k%4) * 4   bytes
__device__ __forceinline__ uint32_t kmajor_off(int row, int k, int rows) {
  return (uint32_t)((k >> 2) * (rows / 8) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D format F32
         | (2u << 7)          // A format TF32
         | (2u << 10)         // B format TF32
         | (0u << 15)         // A K-major
         | (0u << 16)         // B K-major
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void probe(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* a_hi = sm;
  unsigned char* a_lo = a_hi + M * K * 4;
  unsigned char* b_hi = a_lo + M * K * 4;
  unsigned char* b_lo = b_hi + N * K * 4;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = A[i], h = tf32_hi(x);
    *reinterpret_cast<float*>(a_hi + kmajor_off(r, k, M)) = h;
    *reinterpret_cast<float*>(a_lo + kmajor_off(r, k, M)) = x - h;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i], h = tf32_hi(x);
    *reinterpret_cast<float*>(b_hi + kmajor_off(r, k, N)) = h;
    *reinterpret_cast<float*>(b_lo + kmajor_off(r, k, N)) = x - h;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
    const unsigned char* As[3] = {a_hi, a_hi, a_lo};
    const unsigned char* Bs[3] = {b_hi, b_lo, b_hi};
    int n_mma = 0;
    for (int pass = 0; pass < (split ? 3 : 1); ++pass)
      for (int ks = 0; ks < K / 8; ++ks) {
        // one MMA consumes K = 8 tf32 = two 16-B chunks along K, LBO apart
        const uint64_t ad = smem_desc(smem_u32(As[pass]) + ks * 2 * lboA, lboA, 128);
        const uint64_t bd = smem_desc(smem_u32(Bs[pass]) + ks * 2 * lboB, lboB, 128);
        const uint32_t acc = n_mma++ > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMAs (phase 0)
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(&mbar)),
      "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (rows), 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 32 * warp + lane;
    for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
  for (auto& x : B) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  int bad = 0;
  for (int split = 0; split < 2; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    const int smem = 2 * (M * K + N * K) * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, worst = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0, mag = 0;
        for (int k = 0; k < K; ++k) {
          ref += (double)A[i * K + k] * B[j * K + k];
          mag += fabs((double)A[i * K + k] * B[j * K + k]);
        }
        const double d = D[i * N + j] - ref;
        num += d * d;
        den += ref * ref;
        worst = fmax(worst, fabs(d) / mag);
      }
    const double rel = sqrt(num / den);
    printf("{\"split\": %d, \"rel_l2\": %.3e, \"worst_rel_to_abs_sum\": %.3e}\n", split, rel, worst);
    if (rel > (split ? 1e-6 : 2e-3)) bad = 1;
  }
  return bad;
}
