/* A non-Python host driving the C ABI (include/nfgpu.h): build a plan for a small scene,
 * stage a channel subset, run the forward and the adjoint on the GPU, and check both against
 * the operator entry evaluated directly on the host in double precision
 *   A[m,n] = p(f) exp(-j 2 pi f (dT + dR) / c) / (4 pi dT dR),  m = r + R (t + T f).
 * Prints one JSON line; exit status 0 iff relative L2 errors are within the c128 gate (1e-10)
 * and the c64 gate (1e-5). Built by __graft_entry__.build() into examples/abi_demo. */
#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "nfgpu.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define NT 3
#define NR 4
#define NF 5
#define NX 7
#define NY 5
#define NZ 3

static const double C0 = 299792458.0;

static double dist(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return sqrt(dx * dx + dy * dy + dz * dz);
}

static int check(int rc, const char* what) {
  if (rc != NF_OK) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, nf_last_error());
    exit(2);
  }
  return rc;
}

/* one precision: returns the worse of the forward / adjoint relative L2 errors */
static double run(int dtype, const double* tx, const double* rx, const double* freq, const double* pulse,
                  const double* corner, const double* spacing, const int* dims) {
  const int M = NF * NT * NR, N = NX * NY * NZ, B = 23;
  const size_t rs = dtype == NF_C64 ? sizeof(float) : sizeof(double);
  nf_plan* plan;
  check(nf_plan_create(tx, NT, rx, NR, freq, pulse, NF, C0, corner, spacing, dims, 0, NZ, dtype, M, &plan),
        "nf_plan_create");
  /* subset: every second channel from the top, in reverse order (subset order must be respected) */
  int idx[B];
  for (int k = 0; k < B; ++k) idx[k] = (M - 1) - 2 * k;
  double s[2 * N], r[2 * B];
  srand(7);
  for (int i = 0; i < 2 * N; ++i) s[i] = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < 2 * B; ++i) r[i] = rand() / (double)RAND_MAX - 0.5;
  /* host reference */
  double complex yref[B], gref[N];
  for (int n = 0; n < N; ++n) gref[n] = 0;
  for (int k = 0; k < B; ++k) {
    const int m = idx[k], f = m / (NT * NR), t = (m / NR) % NT, rr = m % NR;
    yref[k] = 0;
    for (int n = 0; n < N; ++n) {
      const double v[3] = {corner[0] + (n % NX) * spacing[0], corner[1] + ((n / NX) % NY) * spacing[1],
                           corner[2] + (n / (NX * NY)) * spacing[2]};
      const double dT = dist(v, tx + 3 * t), dR = dist(v, rx + 3 * rr);
      const double complex a = (pulse[2 * f] + I * pulse[2 * f + 1]) *
                               cexp(-I * 2.0 * M_PI * freq[f] * (dT + dR) / C0) / (4.0 * M_PI * dT * dR);
      yref[k] += a * (s[2 * n] + I * s[2 * n + 1]);
      gref[n] += conj(a) * (r[2 * k] + I * r[2 * k + 1]);
    }
  }
  /* device buffers in the plan's precision */
  void *d_s, *d_y, *d_r, *d_g;
  int* d_idx;
  cudaMalloc((void**)&d_idx, sizeof(int) * B);
  cudaMalloc(&d_s, 2 * rs * N);
  cudaMalloc(&d_y, 2 * rs * B);
  cudaMalloc(&d_r, 2 * rs * B);
  cudaMalloc(&d_g, 2 * rs * N);
  cudaMemcpy(d_idx, idx, sizeof(int) * B, cudaMemcpyHostToDevice);
  float sf[2 * N], rf[2 * B];
  for (int i = 0; i < 2 * N; ++i) sf[i] = (float)s[i];
  for (int i = 0; i < 2 * B; ++i) rf[i] = (float)r[i];
  cudaMemcpy(d_s, dtype == NF_C64 ? (void*)sf : (void*)s, 2 * rs * N, cudaMemcpyHostToDevice);
  cudaMemcpy(d_r, dtype == NF_C64 ? (void*)rf : (void*)r, 2 * rs * B, cudaMemcpyHostToDevice);
  check(nf_batch_prepare(plan, d_idx, B, 0), "nf_batch_prepare");
  check(nf_forward(plan, d_s, d_y, 0), "nf_forward");
  check(nf_adjoint(plan, d_r, NULL, d_g, 1.0, 0), "nf_adjoint");
  double y[2 * B], g[2 * N];
  if (dtype == NF_C64) {
    float yf[2 * B], gf[2 * N];
    cudaMemcpy(yf, d_y, sizeof(yf), cudaMemcpyDeviceToHost);
    cudaMemcpy(gf, d_g, sizeof(gf), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 2 * B; ++i) y[i] = yf[i];
    for (int i = 0; i < 2 * N; ++i) g[i] = gf[i];
  } else {
    cudaMemcpy(y, d_y, sizeof(y), cudaMemcpyDeviceToHost);
    cudaMemcpy(g, d_g, sizeof(g), cudaMemcpyDeviceToHost);
  }
  double ny = 0, dy = 0, ng = 0, dg = 0;
  for (int k = 0; k < B; ++k) {
    const double complex e = (y[2 * k] + I * y[2 * k + 1]) - yref[k];
    dy += creal(e * conj(e));
    ny += creal(yref[k] * conj(yref[k]));
  }
  for (int n = 0; n < N; ++n) {
    const double complex e = (g[2 * n] + I * g[2 * n + 1]) - gref[n];
    dg += creal(e * conj(e));
    ng += creal(gref[n] * conj(gref[n]));
  }
  cudaFree(d_idx);
  cudaFree(d_s);
  cudaFree(d_y);
  cudaFree(d_r);
  cudaFree(d_g);
  nf_plan_destroy(plan);
  const double ey = sqrt(dy / ny), eg = sqrt(dg / ng);
  return ey > eg ? ey : eg;
}

int main(void) {
  double tx[3 * NT], rx[3 * NR], freq[NF], pulse[2 * NF];
  for (int t = 0; t < NT; ++t) {
    tx[3 * t] = -0.05 + 0.05 * t;
    tx[3 * t + 1] = 0.04;
    tx[3 * t + 2] = 0.0;
  }
  for (int r = 0; r < NR; ++r) {
    rx[3 * r] = -0.06 + 0.04 * r;
    rx[3 * r + 1] = -0.04;
    rx[3 * r + 2] = 0.0;
  }
  for (int f = 0; f < NF; ++f) {
    freq[f] = 20e9 + 1e9 * f;
    pulse[2 * f] = 1.0 - 0.1 * f;
    pulse[2 * f + 1] = 0.05 * f;
  }
  const double corner[3] = {-0.03, -0.02, 0.28}, spacing[3] = {0.01, 0.01, 0.02};
  const int dims[3] = {NX, NY, NZ};
  const double e128 = run(NF_C128, tx, rx, freq, pulse, corner, spacing, dims);
  const double e64 = run(NF_C64, tx, rx, freq, pulse, corner, spacing, dims);
  printf("{\"c128_rel_l2\": %.3e, \"c64_rel_l2\": %.3e}\n", e128, e64);
  return (e128 <= 1e-10 && e64 <= 1e-5) ? 0 : 1;
}
