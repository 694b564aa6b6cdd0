// peaks.cu — B200 pipe-throughput microbenchmarks for the FP32+SFU roofline
// (MEASURED_PEAKS.json has HBM and bf16 figures only).
//
//   mufu      : sin.approx + cos.approx pairs (MUFU.SIN/COS), 8 independent chains per thread
//   ffma      : scalar FFMA, 8 chains
//   ffma2     : packed FFMA2 (fma.rn.f32x2), 8 chains
//   phasor    : the operator's per-entry phasor math (packed reduce + __sincosf) with no memory,
//               i.e. the entry-rate ceiling of the kernels' instruction mix
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// prints one JSON line with per-SM-per-clock rates and absolute rates at the observed clock.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t as_u64(float2 v) { return *reinterpret_cast<uint64_t*>(&v); }
__device__ __forceinline__ float2 as_f2(uint64_t v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)), "l"(as_u64(c)));
  return as_f2(d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)));
  return as_f2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)));
  return as_f2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)));
  return as_f2(d);
}

__global__ void k_mufu(float* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float s, c;
      asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(x[i]));
      asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(x[i]));
      x[i] = s + c;
    }
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_ffma(float* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i);
  const float a = 0.999f, b = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_ffma2(float* out, int iters, float seed) {
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(seed * (threadIdx.x + i), seed * i);
  const float2 a = make_float2(0.999f, 0.998f), b = make_float2(1e-7f, 2e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], a, b);
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i].x + x[i].y;
  if (acc == 12345.f) out[0] = acc;
}

// per iteration: 8 entries (4 pairs) of the operator's phasor + complex accumulate
__global__ void k_phasor(float* out, int iters, float seed) {
  float2 d[4], h[4], g[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d[i] = make_float2(seed * (threadIdx.x + i), seed * (i + 3));
    h[i] = g[i] = make_float2(0.f, 0.f);
  }
  const float2 M2 = make_float2(12582912.f, 12582912.f);
  float k = 213.0f, base = 0.25f, wr = 0.5f, wi = -0.25f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = fma2(make_float2(k, k), add2(d[i], d[(i + 1) & 3]), make_float2(base, base));
      const float2 f = sub2(x, sub2(add2(x, M2), M2));
      const float2 r = mul2(f, make_float2(6.2831853f, 6.2831853f));
      float2 c, s;
      __sincosf(r.x, &s.x, &c.x);
      __sincosf(r.y, &s.y, &c.y);
      const float2 a = mul2(d[i], c), b = mul2(d[i], s);
      h[i] = fma2(b, make_float2(-wi, -wi), fma2(a, make_float2(wr, wr), h[i]));
      g[i] = fma2(b, make_float2(wr, wr), fma2(a, make_float2(wi, wi), g[i]));
    }
    base += 1e-3f;
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc += h[i].x + h[i].y + g[i].x + g[i].y;
  if (acc == 12345.f) out[0] = acc;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, float* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(d, iters, 1e-3f);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(d, iters, 1e-3f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  float* d;
  cudaMalloc(&d, 64);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  const double nthr = (double)blocks * threads;
  const float t_mufu = run(k_mufu, blocks, threads, iters, d);
  const float t_ffma = run(k_ffma, blocks, threads, iters, d);
  const float t_ffma2 = run(k_ffma2, blocks, threads, iters, d);
  const float t_ph = run(k_phasor, blocks, threads, iters, d);
  const double mufu_s = nthr * iters * 16 / (t_mufu * 1e-3);   // MUFU ops/s
  const double ffma_s = nthr * iters * 8 / (t_ffma * 1e-3);    // FFMA lane-ops/s
  const double ffma2_s = nthr * iters * 16 / (t_ffma2 * 1e-3); // fp32 FMA lane-ops/s (2 per FFMA2)
  const double ph_s = nthr * iters * 8 / (t_ph * 1e-3);        // entries/s
  const double hz = clk_khz * 1e3;
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"mufu_ops_per_s\": %.4e, \"mufu_per_clk_sm_at_attr\": %.2f, "
         "\"ffma_lane_ops_per_s\": %.4e, \"ffma_per_clk_sm_at_attr\": %.1f, \"ffma2_lane_ops_per_s\": %.4e, "
         "\"ffma2_per_clk_sm_at_attr\": %.1f, \"phasor_entries_per_s\": %.4e, \"phasor_entries_per_clk_sm_at_attr\": %.2f, "
         "\"sfu_entry_roof_at_attr\": %.4e}\n",
         sms, hz / 1e6, mufu_s, mufu_s / (sms * hz), ffma_s, ffma_s / (sms * hz), ffma2_s, ffma2_s / (sms * hz), ph_s,
         ph_s / (sms * hz), mufu_s / 2);
  return 0;
}
