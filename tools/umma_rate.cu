// Throughput of tcgen05.mma kind::tf32 (cta_group::1, M = 128, K = 8, A and B from shared memory,
// K-major, no swizzle) as a function of N: every SM issues a long chain of MMAs into one TMEM
// accumulator; the kernel is timed with CUDA events. Prints cycles per MMA per SM and the implied
// dense TF32 rate, one JSON line per N. The values in smem are irrelevant to throughput (zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_rate tools/umma_rate.cu && tools/umma_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (uint64_t)((lbo >> 4) & 0x3FFF) << 16 |
         (uint64_t)((sbo >> 4) & 0x3FFF) << 32 | (uint64_t)1 << 46;
}

__global__ void rate(int n, int iters, int m_rows) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int kbytes = 16 * 4 * 4;  // K = 16 reals per operand row set (two MMAs' worth)
  for (int i = tid; i < (128 + 256) * kbytes / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
                           ((uint32_t)(m_rows >> 4) << 24);
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 128 * kbytes;
    const uint32_t lboA = (m_rows / 8) * 128, lboB = (n / 8) * 128;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t ad = smem_desc(a0 + ks * 2 * lboA, lboA, 128);
        const uint64_t bd = smem_desc(b0 + ks * 2 * lboB, lboB, 128);
        const uint32_t acc = (it | ks) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(&mbar)),
      "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int smem = (128 + 256) * 256;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  const int ms[] = {128, 64};
  const int ns[] = {16, 32, 48, 64, 96, 128, 192, 256};
  for (int m : ms)
    for (int n : ns) {
      rate<<<sms, 128, smem>>>(n, 100, m);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      rate<<<sms, 128, smem>>>(n, iters, m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float msec = 0;
      cudaEventElapsedTime(&msec, e0, e1);
      const cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) {
        printf("{\"m\": %d, \"n\": %d, \"error\": \"%s\"}\n", m, n, cudaGetErrorString(err));
        return 1;
      }
      const double mmas = 2.0 * iters, sec = msec / 1e3;
      const double cyc = sec * clk_khz * 1e3 / mmas;
      const double tflops = 2.0 * m * n * 8 * mmas * sms / sec / 1e12;
      printf("{\"m\": %d, \"n\": %d, \"k\": 8, \"cycles_per_mma\": %.2f, \"tf32_tflops\": %.1f, \"clock_mhz\": %d}\n", m, n,
             cyc, tflops, clk_khz / 1000);
    }
  return 0;
}
