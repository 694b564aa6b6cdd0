// nfgpu.cu — B200 (sm_100a) kernels and C ABI for the SPGM hot path of the
// near-field MIMO imaging reference `nfmimo` (arXiv 2509.00774).
//
// The reference (pkg/src/nfmimo/forward.py:183-336) caches F×(T+R)×N complex128
// phasor tables and turns each forward/adjoint into elementwise products plus
// BLAS dots. Nothing frequency-dependent is stored here. Every operator entry
//     A[m,n] = p_f exp(-j 2π f (dT+dR)/c) / (4π dT dR)            (forward.py:142-155)
// is regenerated in registers. The inputs are a frequency-free per-(antenna, voxel)
// distance table (8 B per pair in c64) and two MUFU ops (sin, cos).
//
// Work decomposition:
//   * voxels are cut into warp tiles of 8×8×4 = 256 voxels (NFGPU_V = 8). Lane L owns 8 voxels
//     that are consecutive in x, held as four fp32x2 pairs so the per-entry arithmetic runs on
//     packed FADD2/FFMA2/FMUL2 (sm_100a).
//   * each tile has an fp64 anchor (its centre). The table stores δ = d − D0(tile, antenna)
//     in fp32, plus 1/d. The per-(channel, tile) phase offset frac(f/c·(D0_T + D0_R))
//     is computed once per channel and tile in fp64. Per entry the phase is
//     x = base + (f/c)·(δT+δR) (|x| ≲ 12 revolutions), fed to MUFU.SIN/COS directly when the plan
//     proves that bound and reduced exactly to [-½, ½] first otherwise: ~1e-6 rad phase error at
//     phases of ~2e3 rad.
//   * the channel batch is sorted on the device by (tx-group, rx, tx, f). Per rx
//     run, a warp keeps the rx-side table entries of its voxels in registers
//     (staged one run ahead with cp.async). Per tx group, the tx-side entries sit in the warp's
//     shared memory. Each entry then costs one conflict-free 16-byte shared load per 4 voxels.
//   * work units are (tile, channel chunk) warps: tile-major with a split tail of shorter chunks
//     when the distance table streams from DRAM, chunk-major with tapered chunks when it stays in L2.
//   * adjoint (+prox): chunks of a tile are combined in fixed order by the last-arriving warp,
//     which also applies the complex soft-threshold prox (solver.py:228-241) and writes the
//     termination statistics (solver.py:244-251). Deterministic, with no float atomics.
//   * forward: per-channel lane partials → warp transpose-reduce through smem every 8 channels →
//     two-level deterministic fp64 column reduce over tiles (or, with a peer communicator, the
//     second level fused with the NVLink all-reduce across voxel-slab ranks).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/nfgpu.h"

namespace {

// Tuning knobs (compile-time; defaults are the measured best on B200).
#ifndef NFGPU_V
#define NFGPU_V 8
#endif
#ifndef NFGPU_TG
#define NFGPU_TG 4
#endif
#ifndef NFGPU_UNROLL
#define NFGPU_UNROLL 2
#endif
#ifndef NFGPU_FWD_WARPS
#define NFGPU_FWD_WARPS 4
#endif
#ifndef NFGPU_ADJ_WARPS
#define NFGPU_ADJ_WARPS 4
#endif
#ifndef NFGPU_TBR
#define NFGPU_TBR 8
#endif
#ifndef NFGPU_MINB_FWD
#define NFGPU_MINB_FWD 4
#endif
#ifndef NFGPU_MINB_ADJ
#define NFGPU_MINB_ADJ 4
#endif
#ifndef NFGPU_FWD_CIS  // c128 forward: 1 = table-based cis_rev, 0 = sincospi (the c64 path ignores it)
#define NFGPU_FWD_CIS false
#endif
#ifndef NFGPU_L2_TABLE_MB  // distance tables up to this size use chunk-major work units (nf_plan::chunk_order)
#define NFGPU_L2_TABLE_MB 256
#endif
#ifndef NFGPU_EXACT_REDUCE
#define NFGPU_EXACT_REDUCE 1
#endif
constexpr int V = NFGPU_V;  // voxels per lane (consecutive in x)
static_assert(V == 4 || V == 8, "V must be 4 or 8");
constexpr int NP = V / 2;  // fp32x2 pairs per lane
constexpr int TILE_X = 8, TILE_Y = V == 8 ? 8 : 4, TILE_Z = 4;
constexpr int TILE = TILE_X * TILE_Y * TILE_Z;  // 32 lanes × V
constexpr int TABW = 2 * TILE;                  // Reals per (tile, antenna): δ block + 1/d block
constexpr int FWD_WARPS = NFGPU_FWD_WARPS;
constexpr int ADJ_WARPS = NFGPU_ADJ_WARPS;
constexpr int TG_MAX = NFGPU_TG;  // tx per shared-memory group
constexpr int UNROLL = NFGPU_UNROLL;
constexpr int TBR = NFGPU_TBR;  // forward transpose depth (channels per lane-reduction)
static_assert(TBR == 8 || TBR == 16, "TBR must be 8 or 16");
// antenna limits per plan (no cap on T + R itself): receivers fit 15 bits of the run key, tx groups 9 bits
constexpr int R_MAX = 32767;
constexpr int TGROUPS_MAX = 511;
constexpr unsigned FULL = 0xffffffffu;
#ifdef NFGPU_DEBUG  // device bounds checks of the CTA-tile kernels (a debug build: tools/build_variants.sh)
#define NF_CHECK(cond, ...)                              \
  do {                                                   \
    if (!(cond)) {                                       \
      printf("NF_CHECK %s:%d: %s | ", __FILE__, __LINE__, #cond); \
      printf(__VA_ARGS__);                               \
      __trap();                                          \
    }                                                    \
  } while (0)
#else
#define NF_CHECK(cond, ...) \
  do {                      \
  } while (0)
#endif

// Programmatic dependent launch: kernels of the SPGM step are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs are scheduled while its
// predecessor drains; each of them waits here before touching its predecessor's outputs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// small kernels let their successor's CTAs be scheduled right away (they wait in pdl_wait());
// the two big kernels keep the implicit trigger at exit so waiting CTAs do not take their SM slots
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
constexpr double PI = 3.14159265358979323846;
constexpr double EXACT_FREE_REV = 12.0;  // largest |phase| (revolutions) fed to MUFU unreduced

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(NF_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------ packed fp32x2 (sm_100a)
__device__ __forceinline__ uint64_t as_u64(float2 v) { return *reinterpret_cast<uint64_t*>(&v); }
__device__ __forceinline__ float2 as_f2(uint64_t v) { return *reinterpret_cast<float2*>(&v); }
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
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)), "l"(as_u64(c)));
  return as_f2(d);
}
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// ------------------------------------------------------------------ V-voxel lane vectors
struct FV {  // the lane's V voxels as NP fp32 pairs: (0,1), (2,3), ...
  float2 p[NP];
};
struct DV {
  double v[V];
};
template <typename Real>
using QV = typename std::conditional<std::is_same<Real, float>::value, FV, DV>::type;

// Lane-data layout in every table row, shared-memory row and staging slot: 16-byte
// quads interleaved across lanes, element (lane L, voxel v) at
//   (v / QUAD) * 32 * QUAD + L * QUAD + v % QUAD,   QUAD = 16 / sizeof(Real),
// so each warp-wide 16-byte load touches 512 contiguous bytes (no bank conflicts).
// `p` points at the lane's first quad (row base + L * QUAD).
__device__ __forceinline__ FV ldv(const float* p) {
  FV q;
#pragma unroll
  for (int i = 0; i < NP / 2; ++i) {
    const float4 t = *reinterpret_cast<const float4*>(p + i * 128);
    q.p[2 * i] = make_float2(t.x, t.y);
    q.p[2 * i + 1] = make_float2(t.z, t.w);
  }
  return q;
}
__device__ __forceinline__ DV ldv(const double* p) {
  DV q;
#pragma unroll
  for (int i = 0; i < V / 2; ++i) {
    const double2 t = *reinterpret_cast<const double2*>(p + i * 64);
    q.v[2 * i] = t.x;
    q.v[2 * i + 1] = t.y;
  }
  return q;
}
__device__ __forceinline__ float get(const FV& q, int v) { return (v & 1) ? q.p[v >> 1].y : q.p[v >> 1].x; }
__device__ __forceinline__ double get(const DV& q, int v) { return q.v[v]; }
__device__ __forceinline__ void zero(FV& q) {
#pragma unroll
  for (int i = 0; i < NP; ++i) q.p[i] = make_float2(0.f, 0.f);
}
__device__ __forceinline__ void zero(DV& q) {
#pragma unroll
  for (int i = 0; i < V; ++i) q.v[i] = 0.0;
}
__device__ __forceinline__ FV make_v(const float* x) {
  FV q;
#pragma unroll
  for (int i = 0; i < NP; ++i) q.p[i] = make_float2(x[2 * i], x[2 * i + 1]);
  return q;
}
__device__ __forceinline__ DV make_v(const double* x) {
  DV q;
#pragma unroll
  for (int i = 0; i < V; ++i) q.v[i] = x[i];
  return q;
}

// fp64 cos/sin(2π·r) for r in [-½, ½] revolutions: (cos, sin) of the nearest 256th of a turn from a
// table, times cos/sin of the remainder |2πδ| <= π/256 by short Taylor polynomials (truncation
// below 1e-20), combined by angle addition. About 14 fp64 operations against ~35 for sincospi; error
// a few ulp (c128 parity is 1e-10).
__device__ double2 g_cis256[256];  // (cos, sin)(2π i / 256), filled by init_cis_kernel
__global__ void init_cis_kernel() {
  double s, c;
  sincospi(threadIdx.x / 128.0, &s, &c);
  g_cis256[threadIdx.x] = make_double2(c, s);
}
__device__ __forceinline__ void cis_rev(double r, double& s, double& c) {
  const double q = rint(r * 256.0);
  const double d = fma(q, -1.0 / 256.0, r) * 6.283185307179586476925;
  const double d2 = d * d;
  const double sd = d * fma(d2, fma(d2, fma(d2, -1.0 / 5040.0, 1.0 / 120.0), -1.0 / 6.0), 1.0);
  const double cd = fma(d2, fma(d2, fma(d2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
  const double2 t = g_cis256[(int)q & 255];
  c = fma(t.x, cd, -t.y * sd);
  s = fma(t.y, cd, t.x * sd);
}

// cos/sin(2π·x_v), x_v = base + k·(dT_v + dR_v), reduced exactly to [-½, ½] revolutions
// (magic-number round-to-nearest, exact for |x| < 2^22) before MUFU.SIN/COS.
//
// EXACT = false (the plan picks it when |x| <= 12 rev is guaranteed): skip the
// explicit reduction and let MUFU.SIN/COS reduce the revolution count. This costs ~1e-6 relative
// precision and saves 3 packed FADDs per voxel pair.
// With EXACT = false the channel record already holds 2π·k and 2π·base (radians), so x is
// the phase in radians and no scaling multiply is needed before __sincosf.
template <bool EXACT, bool CIS_TABLE = true>
__device__ __forceinline__ void phasorv(float k, float base, const FV& dT, const FV& dR, FV& c, FV& s) {
  const float2 M2 = bc(12582912.0f);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const float2 x = fma2(bc(k), add2(dT.p[i], dR.p[i]), bc(base));
    float2 r = x;
    if (EXACT) r = mul2(sub2(x, sub2(add2(x, M2), M2)), bc(6.28318530717958647692f));
    __sincosf(r.x, &s.p[i].x, &c.p[i].x);
    __sincosf(r.y, &s.p[i].y, &c.p[i].y);
  }
}
// CIS_TABLE = false keeps sincospi: the flat forward is LSU-heavy already, and the table gather
// costs it more than the fp64 it saves (c128 forward 3.0e11 -> 2.8e11 with it; adjoint 2.6e11 -> 3.0e11)
template <bool EXACT, bool CIS_TABLE = true>
__device__ __forceinline__ void phasorv(double k, double base, const DV& dT, const DV& dR, DV& c, DV& s) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double x = fma(k, dT.v[v] + dR.v[v], base);
    if (CIS_TABLE)
      cis_rev(x - rint(x), s.v[v], c.v[v]);
    else
      sincospi(2.0 * (x - rint(x)), &s.v[v], &c.v[v]);
  }
}

// adjoint: h += iT·e^{+jθ}·w  (w = conj(p)/(4π)·r, one complex per channel)
__device__ __forceinline__ void adj_acc(const FV& iT, const FV& c, const FV& s, float wr, float wi, FV& hr, FV& hi) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const float2 a = mul2(iT.p[i], c.p[i]), b = mul2(iT.p[i], s.p[i]);
    hr.p[i] = fma2(b, bc(-wi), fma2(a, bc(wr), hr.p[i]));
    hi.p[i] = fma2(b, bc(wr), fma2(a, bc(wi), hi.p[i]));
  }
}
__device__ __forceinline__ void adj_acc(const DV& iT, const DV& c, const DV& s, double wr, double wi, DV& hr,
                                        DV& hi) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double a = iT.v[v] * c.v[v], b = iT.v[v] * s.v[v];
    hr.v[v] = fma(-b, wi, fma(a, wr, hr.v[v]));
    hi.v[v] = fma(b, wr, fma(a, wi, hi.v[v]));
  }
}
// end of an rx run: g += iR·h, h = 0
__device__ __forceinline__ void flush(const FV& iR, FV& hr, FV& hi, FV& gr, FV& gi) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    gr.p[i] = fma2(iR.p[i], hr.p[i], gr.p[i]);
    gi.p[i] = fma2(iR.p[i], hi.p[i], gi.p[i]);
    // h = 0 as one packed multiply per pair (h is finite; a literal 0 costs two 32-bit moves)
    hr.p[i] = mul2(hr.p[i], bc(0.f));
    hi.p[i] = mul2(hi.p[i], bc(0.f));
  }
}
__device__ __forceinline__ void flush(const DV& iR, DV& hr, DV& hi, DV& gr, DV& gi) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    gr.v[v] = fma(iR.v[v], hr.v[v], gr.v[v]);
    gi.v[v] = fma(iR.v[v], hi.v[v], gi.v[v]);
  }
  zero(hr);
  zero(hi);
}
// forward: ŝ = iR·s for the current rx run, and −Re ŝ (the subtracted term of Im, kept per run)
__device__ __forceinline__ void scale_s(const FV& iR, const FV& sr, const FV& si, FV& shr, FV& shi, FV& nshr) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    shr.p[i] = mul2(iR.p[i], sr.p[i]);
    shi.p[i] = mul2(iR.p[i], si.p[i]);
    nshr.p[i] = mul2(shr.p[i], bc(-1.f));
  }
}
__device__ __forceinline__ void scale_s(const DV& iR, const DV& sr, const DV& si, DV& shr, DV& shi, DV& nshr) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    shr.v[v] = iR.v[v] * sr.v[v];
    shi.v[v] = iR.v[v] * si.v[v];
    nshr.v[v] = -shr.v[v];
  }
}
// forward: Σ_v iT·e^{-jθ}·ŝ over the lane's V voxels
__device__ __forceinline__ float2 fwd_part(const FV& iT, const FV& c, const FV& s, const FV& shr, const FV& shi,
                                           const FV& nshr) {
  float2 pr = make_float2(0.f, 0.f), pi = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const float2 a = mul2(iT.p[i], c.p[i]), b = mul2(iT.p[i], s.p[i]);
    pr = fma2(b, shi.p[i], fma2(a, shr.p[i], pr));
    pi = fma2(b, nshr.p[i], fma2(a, shi.p[i], pi));
  }
  return make_float2(pr.x + pr.y, pi.x + pi.y);
}
__device__ __forceinline__ double2 fwd_part(const DV& iT, const DV& c, const DV& s, const DV& shr, const DV& shi,
                                            const DV& nshr) {
  double pr = 0, pi = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double a = iT.v[v] * c.v[v], b = iT.v[v] * s.v[v];
    pr = fma(b, shi.v[v], fma(a, shr.v[v], pr));
    pi = fma(b, nshr.v[v], fma(a, shi.v[v], pi));
  }
  return make_double2(pr, pi);
}

template <typename Real>
struct Real2T;
template <>
struct Real2T<float> {
  using T = float2;
};
template <>
struct Real2T<double> {
  using T = double2;
};
template <typename Real>
using R2 = typename Real2T<Real>::T;
template <typename Real>
struct Real4T;
template <>
struct Real4T<float> {
  using T = float4;
};
template <>
struct Real4T<double> {
  struct T {
    double x, y, z, w;
  };
};
template <typename Real>
using R4 = typename Real4T<Real>::T;

// ------------------------------------------------------------------ geometry
struct Geo {
  int T, R, A, F;
  int nx, ny, nzs, zb;  // slab: nzs planes starting at global plane zb
  int ntx, nty, ntz, ntiles;
  int Tg, ng;
  int tg_mul;  // ceil(65536 / Tg): tx group of transmitter t = (t * tg_mul) >> 16 (exact for t < 32768 / Tg)
  double corner[3], sp[3];
};
__device__ __forceinline__ int tx_group(const Geo& g, int t) { return (t * g.tg_mul) >> 16; }

__device__ __forceinline__ void tile_coords(const Geo& g, int tile, int& tx, int& ty, int& tz) {
  tz = tile / (g.ntx * g.nty);
  const int rem = tile - tz * g.ntx * g.nty;
  ty = rem / g.ntx;
  tx = rem - ty * g.ntx;
}

// V = 8: lane L of tile (tx,ty,tz) owns x = 8tx + v (v < 8), y = 8ty + (L&7), z = 4tz + (L>>3)
// V = 4: x = 8tx + 4(L&1) + v, y = 4ty + ((L>>1)&3), z = 4tz + (L>>3)
__device__ __forceinline__ void lane_voxel(int tx, int ty, int tz, int L, int& x0, int& y, int& z) {
  if (V == 8) {
    x0 = tx * TILE_X;
    y = ty * TILE_Y + (L & 7);
  } else {
    x0 = tx * TILE_X + (L & 1) * V;
    y = ty * TILE_Y + ((L >> 1) & 3);
  }
  z = tz * TILE_Z + (L >> 3);
}

// table[tile][a][2][32][V]: [0] = δ = d − D0, [1] = 1/d for the lane's V voxels; D0[tile][a] in fp64.
template <typename Real>
__global__ void build_table_kernel(Geo g, const double* __restrict__ ant, Real* __restrict__ tab,
                                   double* __restrict__ D0) {
  const int tile = blockIdx.x, a = blockIdx.y, L = threadIdx.x;
  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  const double px = ant[3 * a], py = ant[3 * a + 1], pz = ant[3 * a + 2];
  const double ax = g.corner[0] + (tx * TILE_X + 0.5 * (TILE_X - 1)) * g.sp[0];
  const double ay = g.corner[1] + (ty * TILE_Y + 0.5 * (TILE_Y - 1)) * g.sp[1];
  const double az = g.corner[2] + (g.zb + tz * TILE_Z + 0.5 * (TILE_Z - 1)) * g.sp[2];
  const double d0 = sqrt((ax - px) * (ax - px) + (ay - py) * (ay - py) + (az - pz) * (az - pz));
  if (L == 0) D0[(size_t)tile * g.A + a] = d0;
  int x0, y, z;
  lane_voxel(tx, ty, tz, L, x0, y, z);
  Real* out = tab + ((size_t)tile * g.A + a) * TABW;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int x = x0 + v;
    Real dl = 0, iv = 0;
    if (x < g.nx && y < g.ny && z < g.nzs) {
      // voxel centre exactly as geometry.voxel_centers (geometry.py:194-207)
      const double cx = g.corner[0] + x * g.sp[0];
      const double cy = g.corner[1] + y * g.sp[1];
      const double cz = g.corner[2] + (g.zb + z) * g.sp[2];
      const double d = sqrt((cx - px) * (cx - px) + (cy - py) * (cy - py) + (cz - pz) * (cz - pz));
      dl = (Real)(d - d0);
      iv = (Real)(1.0 / d);
    }
    constexpr int QD = 16 / (int)sizeof(Real);
    const int o = (v / QD) * 32 * QD + L * QD + v % QD;
    out[o] = dl;
    out[TILE + o] = iv;
  }
}

// ------------------------------------------------------------------ batch prep
// Sort key of a channel: (tx group, rx, tx in group, f) -- runs of one receiver within one tx group, whose tx rows a
// warp stages -- or, for the CTA-tile kernels (all rows resident), rx-major (rx, tx group, tx in group, f): a
// receiver's rows (and the forward's scaled iterate, the adjoint's partial sum) then change once per receiver.
struct KeyMap {
  int T, R, F, Tg, ng, rxmajor;
};
__device__ __forceinline__ int key_of(const KeyMap& k, int m) {
  const int TR = k.T * k.R;
  const int f = m / TR;
  const int rem = m - f * TR;
  const int t = rem / k.R;
  const int r = rem - t * k.R;
  const int tg = t / k.Tg, tl = t - tg * k.Tg;
  const int outer = k.rxmajor ? r * k.ng + tg : tg * k.R + r;
  return (outer * k.Tg + tl) * k.F + f;
}
__device__ __forceinline__ int4 chan_of_key(const KeyMap& k, int key) {  // {f, t, r, tg}
  const int f = key % k.F;
  int q = key / k.F;
  const int tl = q % k.Tg;
  q /= k.Tg;
  int r, tg;
  if (k.rxmajor) {
    tg = q % k.ng;
    r = q / k.ng;
  } else {
    r = q % k.R;
    tg = q / k.R;
  }
  return make_int4(f, tg * k.Tg + tl, r, tg);
}

__global__ void mark_kernel(KeyMap km, const int* __restrict__ idx, int B, int* __restrict__ pos_of_key) {
  pdl_wait_and_release();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) pos_of_key[key_of(km, idx[i])] = i;
}

__device__ __forceinline__ int block_excl_scan_1024(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;
  }
  __syncthreads();
  total = sh[31];
  const int pre = (wid > 0 ? sh[wid - 1] : 0) + x - v;
  __syncthreads();
  return pre;
}

// exclusive block scan for any blockDim that is a multiple of 32 (<= 1024); sh: 32 ints of shared memory
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;
  }
  __syncthreads();
  total = sh[nw - 1];
  const int res = (wid > 0 ? sh[wid - 1] : 0) + x - v;
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(1024) count_kernel(const int* __restrict__ pos_of_key, int KS,
                                                      int* __restrict__ cnt) {
  pdl_wait_and_release();
  const int key = blockIdx.x * 1024 + threadIdx.x;
  const int f = (key < KS && pos_of_key[key] >= 0) ? 1 : 0;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) scan_kernel(int* __restrict__ cnt, int n) {
  pdl_wait_and_release();
  __shared__ int sh[32];
  int carry = 0;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? cnt[i] : 0;
    int total;
    const int pre = block_excl_scan_1024(v, sh, total);
    if (i < n) cnt[i] = carry + pre;
    carry += total;
  }
}

// Per sorted position: everything a warp needs about a channel except its tile-dependent
// phase offset. pk = t | r << 16 (T <= 65535, R <= R_MAX); the tx group is t / Tg.
struct ChanRec {
  double kd;  // f / c (fp64, for the anchor phase)
  float kf;   // f / c (fp32, per-entry slope)
  int pk;
};
__device__ __forceinline__ int pk_t(int pk) { return pk & 0xffff; }
__device__ __forceinline__ int pk_r(int pk) { return pk >> 16; }

// sorted position j <- key order; crec[j], sf[j] = f
__global__ void __launch_bounds__(1024) compact_kernel(KeyMap km, int* __restrict__ pos_of_key, int KS,
                                                        const int* __restrict__ off, int* __restrict__ sm,
                                                        int* __restrict__ spos, ChanRec* __restrict__ crec,
                                                        int* __restrict__ sf, const double* __restrict__ kd) {
  pdl_wait_and_release();
  __shared__ int sh[32];
  const int key = blockIdx.x * 1024 + threadIdx.x;
  const int p = key < KS ? pos_of_key[key] : -1;
  int total;
  const int pre = block_excl_scan_1024(p >= 0 ? 1 : 0, sh, total);
  if (p >= 0) {
    const int j = off[blockIdx.x] + pre;
    const int4 c = chan_of_key(km, key);
    sm[j] = c.z + km.R * (c.y + km.T * c.x);
    spos[j] = p;
    ChanRec q;
    q.kd = kd[c.x];
    q.kf = (float)q.kd;
    q.pk = c.y | (c.z << 16);
    crec[j] = q;
    sf[j] = c.x;
    pos_of_key[key] = -1;
  }
}

// ------------------------------------------------------------------ sampler
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t feistel(uint32_t x, int hb, uint64_t key) {
  const uint32_t mask = (1u << hb) - 1u;
  uint32_t l = x >> hb, r = x & mask;
#pragma unroll
  for (int round = 0; round < 6; ++round) {
    const uint32_t k = (uint32_t)(key >> ((round & 1) ? 32 : 0)) ^ (0x9e3779b9u * (round + 1));
    const uint32_t f = hash32(r ^ k) & mask;
    const uint32_t nl = r;
    r = l ^ f;
    l = nl;
  }
  return (l << hb) | r;
}
__host__ __device__ __forceinline__ uint64_t sample_key(uint64_t seed, uint64_t iter) {
  return (seed * 0x9E3779B97F4A7C15ULL) ^ (iter * 0xD1B54A32D192ED03ULL) ^ 0x2545F4914F6CDD1DULL;
}
// iter_dev != null: the iteration number is read from device memory (graph-capturable loop)
__global__ void sample_kernel(uint64_t seed, uint64_t iter, const unsigned long long* __restrict__ iter_dev, int hb,
                              int M, int B, int* __restrict__ idx) {
  pdl_wait_and_release();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B) return;
  const uint64_t key = sample_key(seed, iter_dev ? (uint64_t)*iter_dev : iter);
  uint32_t x = (uint32_t)j;
  do {
    x = feistel(x, hb, key);
  } while (x >= (uint32_t)M);
  idx[j] = (int)x;
}
__global__ void bump_kernel(unsigned long long* it) {
  pdl_wait_and_release();
  *it += 1ULL;
}

// Structured (Cartesian) sampler on the device: k_a distinct sorted indices out of n_a for each axis
// a in {frequency, tx, rx}, the first k_a images of a keyed Feistel permutation of [0, n_a)
// (cycle-walking on the next even power of two), ranked into ascending order. One block of 256
// threads; lists go to out = [F | T | R] (the plan's structured-batch lists). iter_dev: the
// iteration number is read from (and then advanced in) device memory, so the call is capturable.
__global__ void __launch_bounds__(256) struct_sample_kernel(uint64_t seed, uint64_t iter,
                                                            unsigned long long* __restrict__ iter_dev, int F, int T,
                                                            int R, int nf, int nt, int nr, int* __restrict__ out) {
  __shared__ int vals[256];
  const uint64_t key0 = sample_key(seed, iter_dev ? (uint64_t)*iter_dev : iter);
  const int ns[3] = {F, T, R}, ks[3] = {nf, nt, nr}, offs[3] = {0, F, F + T};
  for (int axis = 0; axis < 3; ++axis) {
    const int n = ns[axis], k = ks[axis];
    int bits = 2;
    while ((1 << bits) < n) bits += 2;
    const uint64_t key = key0 ^ (0x632BE59BD9B4E019ULL * (uint64_t)(axis + 1));
    for (int i = threadIdx.x; i < k; i += 256) {
      uint32_t x = (uint32_t)i;
      do {
        x = feistel(x, bits / 2, key);
      } while (x >= (uint32_t)n);
      vals[i] = (int)x;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += 256) {  // rank of vals[i] among the k distinct values
      const int v = vals[i];
      int pos = 0;
      for (int j = 0; j < k; ++j) pos += vals[j] < v;
      out[offs[axis] + pos] = v;
    }
    __syncthreads();
  }
  if (iter_dev && threadIdx.x == 0) *iter_dev += 1ULL;  // every thread has read it
}
__global__ void set_kernel(unsigned long long* it, unsigned long long v) { *it = v; }

// ------------------------------------------------------------------ per-warp shared state
template <typename Real>
struct WarpSmem {
  Real* tside;    // [Tg][2][32][V] tx-side rows of the current tx group
  Real* rslot;    // [2][2][32][V] rx-side rows, ping-pong staging (cp.async)
  double* d0;     // [A]
  R4<Real>* rec;  // [34] {k, base, wr, wi}
  int2* rect;     // [34] {tside offset, run key}
};
__host__ __device__ constexpr int d0_slots(int A) { return (A + 1) & ~1; }  // keep 16-byte alignment
template <typename Real>
__host__ __device__ constexpr size_t warp_smem_bytes(int Tg, int A, int nslots = 2) {
  return (size_t)(Tg + nslots) * TABW * sizeof(Real) + (size_t)d0_slots(A) * sizeof(double) +
         34 * sizeof(R4<Real>) + 34 * sizeof(int2);
}
template <typename Real>
__device__ __forceinline__ WarpSmem<Real> carve(unsigned char* base, int Tg, int A, int nslots = 2) {
  WarpSmem<Real> ws;
  ws.tside = reinterpret_cast<Real*>(base);
  ws.rslot = ws.tside + (size_t)Tg * TABW;
  ws.d0 = reinterpret_cast<double*>(base + (size_t)(Tg + nslots) * TABW * sizeof(Real));
  ws.rec = reinterpret_cast<R4<Real>*>(reinterpret_cast<unsigned char*>(ws.d0) + d0_slots(A) * sizeof(double));
  ws.rect = reinterpret_cast<int2*>(ws.rec + 34);
  return ws;
}

// Stage receiver r's rows for this lane's voxels into a shared slot with per-lane cp.async
// (LDGSTS): each lane copies and later reads back only its own 2·V Reals, so no warp sync
// is needed, only cp.async.wait_all by the same lane.
template <typename Real>
__device__ __forceinline__ void stage_rx(const Geo& g, const Real* __restrict__ tabt, int r, Real* slot, int L) {
  constexpr int QD = 16 / (int)sizeof(Real);
  const Real* src = tabt + (size_t)(g.T + r) * TABW + L * QD;
  Real* dst = slot + L * QD;
  constexpr int n16 = V / QD;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < n16; ++i) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + h * TILE + i * 32 * QD);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + h * TILE + i * 32 * QD)
                   : "memory");
    }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Rows of receiver rr for the run that starts now: from the ping-pong slot if it was
// prefetched, else straight from global. Then prefetch the next receiver (wrapping to 0,
// the first receiver of the next tx group) into the other slot.
template <typename Real>
__device__ __forceinline__ void rx_run_rows(const Geo& g, const Real* __restrict__ tabt, const WarpSmem<Real>& ws,
                                            int rr, int& pf_r, int& slot, int L, QV<Real>& dR, QV<Real>& iR) {
  if (rr != pf_r) {  // not prefetched: drain any stale prefetch into this slot, then stage rr
    stage_wait();
    stage_rx<Real>(g, tabt, rr, ws.rslot + (size_t)slot * TABW, L);
  }
  stage_wait();
  __syncwarp();  // a tx-group copy issued at this run start is complete for every lane
  const Real* sl = ws.rslot + (size_t)slot * TABW + L * (16 / (int)sizeof(Real));
  dR = ldv(sl);
  iR = ldv(sl + TILE);
  slot ^= 1;
  pf_r = rr + 1 < g.R ? rr + 1 : 0;
  stage_rx<Real>(g, tabt, pf_r, ws.rslot + (size_t)slot * TABW, L);
}

// Start copying the tx-side table rows of tx group tg for this tile into the warp's smem
// (cp.async, no wait). The caller's stage_wait() + __syncwarp() completes it, overlapped
// with the rx-row staging of the same run start.
template <typename Real>
__device__ __forceinline__ void load_tgroup_async(const Geo& g, const Real* __restrict__ tabt, Real* tside, int tg,
                                                  int L) {
  const int ta = tg * g.Tg;
  const int nt = min(g.Tg, g.T - ta);
  const char* src = reinterpret_cast<const char*>(tabt + (size_t)ta * TABW);
  const unsigned dst = (unsigned)__cvta_generic_to_shared(tside);
  const int n = nt * TABW * (int)sizeof(Real) / 16;
  __syncwarp();  // every lane is done reading the previous group
  for (int i = L; i < n; i += 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * i), "l"(src + 16 * (size_t)i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <typename Real>
__device__ __forceinline__ Real int_bits(int v);
template <>
__device__ __forceinline__ float int_bits<float>(int v) { return __int_as_float(v); }
template <>
__device__ __forceinline__ double int_bits<double>(int v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ int bits_int(float v) { return __float_as_int(v); }
__device__ __forceinline__ int bits_int(double v) { return (int)__double_as_longlong(v); }

__device__ __forceinline__ float with_low2(float v, int k) { return __int_as_float((__float_as_int(v) & ~3) | k); }
__device__ __forceinline__ double with_low2(double v, int k) {
  return __longlong_as_double((__double_as_longlong(v) & ~3LL) | k);
}
__device__ __forceinline__ int low2(float v) { return __float_as_int(v) & 3; }
__device__ __forceinline__ int low2(double v) { return (int)(__double_as_longlong(v) & 3LL); }

// Build the 32 channel records of one batch (lane L <-> sorted position jb+L) from the
// prefetched ChanRec/w in registers, and prefetch the next batch's. Returns the bitmask of
// run starts (a run = maximal stretch with equal (rx, tx group)). rect[L] = {tx-row offset in the
// group, rx | tx group << 16 | run end << 24}; the run end of position L is the next run start
// after L (or nb), so the channel loops read their segment bound with the same shared load.
template <typename Real, bool EXACT>
__device__ __forceinline__ unsigned build_records(const Geo& g, const WarpSmem<Real>& ws,
                                                  const ChanRec* __restrict__ crec,
                                                  const R2<Real>* __restrict__ wrec, int jb, int nb, int jend,
                                                  int L, int& carry, ChanRec& nxt, R2<Real>& nxtw) {
  const ChanRec cr = nxt;
  const R2<Real> w = nxtw;
  if (jb + 32 + L < jend) {
    nxt = crec[jb + 32 + L];
    if (wrec) nxtw = wrec[jb + 32 + L];
  }
  int key = -1, toff = 0;
  if (L < nb) {
    const int t = pk_t(cr.pk), r = pk_r(cr.pk), tg = tx_group(g, t);
    const double x = cr.kd * (ws.d0[t] + ws.d0[g.T + r]);
    R4<Real> q;
    if constexpr (std::is_same<Real, float>::value) {
      if (EXACT) {
        q.x = cr.kf;
        q.y = (float)(x - rint(x));
      } else {  // radians: slope 2π f/c and offset 2π frac(...)
        q.x = (float)(2.0 * PI * cr.kd);
        q.y = (float)(2.0 * PI * (x - rint(x)));
      }
    } else {
      q.x = cr.kd;
      q.y = (Real)(x - rint(x));
    }
    toff = (t - tg * g.Tg) * TABW;
    if (wrec) {
      q.z = w.x;
      q.w = w.y;
      // adjoint: the tx index within the group (< TG_MAX = 4) rides in the 2 low bits of the phase offset
      // (≤ 3 ulp of |base| ≤ π: < 1e-6 rad), so one broadcast load per channel brings the whole record
      q.y = with_low2(q.y, t - tg * g.Tg);
    } else {  // forward: the tx-row offset rides in .z as a bit pattern (one broadcast load per channel)
      q.z = int_bits<Real>(toff);
      q.w = 0;
    }
    ws.rec[L] = q;
    key = r | (tg << 15);  // run key: rx (15 bits) | tx group (9 bits); the run end rides in bits 24-29
  }
  int prev = __shfl_up_sync(FULL, key, 1);
  if (L == 0) prev = carry;
  const unsigned starts = __ballot_sync(FULL, L < nb && key != prev);
  carry = __shfl_sync(FULL, key, nb - 1);
  if (L < nb) {
    const unsigned later = L < 31 ? (starts >> (L + 1)) << (L + 1) : 0u;
    const int end = later ? __ffs(later) - 1 : nb;
    ws.rect[L] = make_int2(toff, key | (end << 24));
  }
  __syncwarp();
  return starts;
}

template <typename Real>
__device__ __forceinline__ void prefetch_first(const ChanRec* __restrict__ crec, const R2<Real>* __restrict__ wrec,
                                               int j0, int j1, int L, ChanRec& nxt, R2<Real>& nxtw) {
  nxt.kd = 0;
  nxt.kf = 0;
  nxt.pk = 0;
  nxtw.x = 0;
  nxtw.y = 0;
  if (j0 + L < j1) {
    nxt = crec[j0 + L];
    if (wrec) nxtw = wrec[j0 + L];
  }
}

// ------------------------------------------------------------------ adjoint (+prox)
// Boundary c of C channel chunks over n channels. order 0: equal chunks. order 1: sizes fall
// linearly, g(x) = (x − h·x²)/(1 − h) (monotone for h < ½, g(1) = 1; the last chunk is 1 − 2h of the
// first), so that with chunk-major unit order the last wave of a launch is made of the smallest chunks.
__device__ __forceinline__ int chunk_bound(int n, int c, int C, int order, float h) {
  if (order == 0 || c >= C) return (int)(((long long)n * c) / C);
  const double x = (double)c / C;
  return (int)((double)n * ((x - h * x * x) / (1.0 - h)));
}
// (tile, chunk) of a warp work unit: tile-major (a tile's chunks adjacent, sharing its table rows
// in L2) or chunk-major (tables that stay in L2: with tapered chunks the launch ends on short units)
__device__ __forceinline__ void unit_coords(int unit, int ntiles, int C, int order, int& tile, int& chunk) {
  if (order == 0) {
    tile = unit / C;
    chunk = unit - tile * C;
  } else {
    chunk = unit / ntiles;
    tile = unit - chunk * ntiles;
  }
}
// Units of a launch: chunk-major (order 1) as unit_coords, or tile-major with a split tail: tiles [0, t1)
// in C chunks, tiles [t1, ntiles) in C2 (shorter) chunks, so the last wave of the launch is made of short
// units while every tile's chunks stay adjacent (table rows reused from L2). Ct = chunk count of the tile.
__device__ __forceinline__ void unit_map(int unit, int ntiles, int C, int t1, int C2, int order, int& tile, int& chunk,
                                         int& Ct) {
  if (order != 0) {
    unit_coords(unit, ntiles, C, order, tile, chunk);
    Ct = C;
    return;
  }
  const int u1 = t1 * C;
  if (unit < u1) {
    tile = unit / C;
    chunk = unit - tile * C;
    Ct = C;
  } else {
    const int k = (unit - u1) / C2;
    tile = t1 + k;
    chunk = unit - u1 - k * C2;
    Ct = C2;
  }
}

template <typename Real>
struct AdjArgs {
  Geo g;
  const Real* __restrict__ tab;
  const double* __restrict__ D0;
  const ChanRec* __restrict__ crec;
  const R2<Real>* __restrict__ wrec;
  int B, CH;
  int order;                 // unit order: 0 tile-major, equal chunks; 1 chunk-major, tapered (chunk_bound)
  int t1, CH2;               // tile-major tail: tiles [t1, ntiles) in CH2 chunks (unit_map; t1 = ntiles: none)
  float taper;               // chunk-major taper coefficient h (chunk_bound)
  Real* __restrict__ gpart;  // [CH][ntiles][32][4] complex (CH > 1)
  int* __restrict__ cnt;     // [ntiles] arrival counters (zero between launches)
  // plain adjoint
  Real* __restrict__ gout;
  double scale;
  // prox
  const Real* __restrict__ s_in;
  Real* __restrict__ s_out;
  double eta_over_b, alpha;
  double* __restrict__ stat_part;  // [ntiles][4]
};

// w_j = conj(p_f)/(4π)·(r[spos_j] − ymeas[m_j]) in sorted order; dpart[block] = Σ |r − y|²
template <typename Real>
__global__ void __launch_bounds__(256) resid_kernel(const int* __restrict__ sm, const int* __restrict__ spos,
                                                    const int* __restrict__ sf, int B,
                                                    const Real* __restrict__ r, const Real* __restrict__ ymeas,
                                                    const double* __restrict__ pulse, R2<Real>* __restrict__ wrec,
                                                    double* __restrict__ dpart) {
  pdl_wait_and_release();
  __shared__ double sh[8];
  const int j = blockIdx.x * 256 + threadIdx.x;
  double e = 0;
  if (j < B) {
    const int k = spos[j];
    double rr = (double)r[2 * (size_t)k], ri = (double)r[2 * (size_t)k + 1];
    if (ymeas) {
      const int m = sm[j];
      rr -= (double)ymeas[2 * (size_t)m];
      ri -= (double)ymeas[2 * (size_t)m + 1];
    }
    e = rr * rr + ri * ri;
    const int f = sf[j];
    const double pr = pulse[2 * f] / (4.0 * PI), pim = -pulse[2 * f + 1] / (4.0 * PI);
    R2<Real> w;
    w.x = (Real)(pr * rr - pim * ri);
    w.y = (Real)(pr * ri + pim * rr);
    wrec[j] = w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int i = 0; i < 8; ++i) t += sh[i];
    dpart[blockIdx.x] = t;
  }
}

// Adjoint epilogue shared by the flat and structured kernels: publish this (tile, chunk)
// partial; the last of the tile's CH warps sums the partials in chunk order and writes
// g (plain adjoint) or applies the prox and the termination statistics (SPGM step).
// LOOP (spgm_loop_kernel): the iterate is read through L2 (another SM wrote it an iteration ago)
template <typename Real, bool PROX, bool LOOP = false>
__device__ __forceinline__ void adj_epilogue(const AdjArgs<Real>& a, int tile, int chunk, int C, int L, const QV<Real>& gr,
                                             const QV<Real>& gi, const Real* __restrict__ s_in,
                                             Real* __restrict__ s_out) {
  const Geo& g = a.g;
  Real Gr[V], Gi[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    Gr[v] = get(gr, v);
    Gi[v] = get(gi, v);
  }
  if (C > 1) {
    // publish this chunk's partial (the lane's 2V Reals, interleaved re/im, as 16-byte stores); the last of
    // the C warps of this tile combines in chunk order, four chunks' loads in flight at a time
    using U16 = typename std::conditional<std::is_same<Real, float>::value, float4, double2>::type;
    constexpr int NU = 2 * V * (int)sizeof(Real) / 16;
    constexpr int PU = 16 / (int)sizeof(Real);  // Reals per U16
    U16* mine = reinterpret_cast<U16*>(a.gpart + (((size_t)chunk * g.ntiles + tile) * 32 + L) * (2 * V));
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      Real t[PU];
#pragma unroll
      for (int k = 0; k < PU; ++k) t[k] = ((u * PU + k) & 1) ? Gi[(u * PU + k) >> 1] : Gr[(u * PU + k) >> 1];
      mine[u] = *reinterpret_cast<const U16*>(t);
    }
    __threadfence();
    int last = 0;
    if (L == 0) last = atomicAdd(a.cnt + tile, 1) == C - 1;
    last = __shfl_sync(FULL, last, 0);
    if (!last) return;
    __threadfence();
#pragma unroll
    for (int v = 0; v < V; ++v) Gr[v] = Gi[v] = 0;
#pragma unroll 4
    for (int ch = 0; ch < C; ++ch) {
      const U16* q = reinterpret_cast<const U16*>(a.gpart + (((size_t)ch * g.ntiles + tile) * 32 + L) * (2 * V));
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const U16 w = __ldcg(q + u);
        const Real* t = reinterpret_cast<const Real*>(&w);
#pragma unroll
        for (int k = 0; k < PU; ++k) {
          const int e = u * PU + k;
          if (e & 1)
            Gi[e >> 1] += t[k];
          else
            Gr[e >> 1] += t[k];
        }
      }
    }
    if (L == 0) a.cnt[tile] = 0;
  }

  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(tx, ty, tz, L, x0, y, z);
  double st0 = 0, st1 = 0, st3 = 0;
  // The lane's V voxels are consecutive in x: when all are inside the grid (and 16-byte aligned), its
  // iterate is read and its new iterate (or gradient) written as 16-byte vectors, else voxel by voxel.
  using U16 = typename std::conditional<std::is_same<Real, float>::value, float4, double2>::type;
  constexpr int NU = 2 * V * (int)sizeof(Real) / 16;
  const bool full = x0 + V <= g.nx && y < g.ny && z < g.nzs && (sizeof(Real) == 8 || (g.nx & 1) == 0);
  const size_t n0 = ((size_t)z * g.ny + y) * g.nx + x0;
  Real io[2 * V];  // interleaved (re, im): s_in in, s_out (or g) out
  if (PROX) {
    if (full) {
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if constexpr (LOOP)
          *reinterpret_cast<U16*>(io + u * (16 / sizeof(Real))) = __ldcg(reinterpret_cast<const U16*>(s_in + 2 * n0) + u);
        else
          *reinterpret_cast<U16*>(io + u * (16 / sizeof(Real))) = reinterpret_cast<const U16*>(s_in + 2 * n0)[u];
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool in = x0 + v < g.nx && y < g.ny && z < g.nzs;
        if constexpr (LOOP) {
          io[2 * v] = in ? __ldcg(s_in + 2 * (n0 + v)) : Real(0);
          io[2 * v + 1] = in ? __ldcg(s_in + 2 * (n0 + v) + 1) : Real(0);
        } else {
          io[2 * v] = in ? s_in[2 * (n0 + v)] : Real(0);
          io[2 * v + 1] = in ? s_in[2 * (n0 + v) + 1] : Real(0);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (!(x0 + v < g.nx && y < g.ny && z < g.nzs)) continue;
    if (!PROX) {
      io[2 * v] = (Real)(a.scale * Gr[v]);
      io[2 * v + 1] = (Real)(a.scale * Gi[v]);
    } else {
      const Real s_r = io[2 * v], s_i = io[2 * v + 1];
      const Real ur = s_r - (Real)a.eta_over_b * Gr[v];
      const Real ui = s_i - (Real)a.eta_over_b * Gi[v];
      const Real mag = hypot(ur, ui);  // |u| as np.abs (no overflow / underflow of the squares)
      const Real al = (Real)a.alpha;
      const Real sc = mag > al ? (mag - al) / mag : Real(0);
      const Real o_r = ur * sc, o_i = ui * sc;
      io[2 * v] = o_r;
      io[2 * v + 1] = o_i;
      // |s|, |o| in fp64: for c64 inputs the squares cannot overflow or underflow, so sqrt is as exact as hypot
      const double m0 = sizeof(Real) == 4 ? sqrt(fma((double)s_r, (double)s_r, (double)s_i * (double)s_i))
                                          : hypot((double)s_r, (double)s_i);
      const double m1 = sizeof(Real) == 4 ? sqrt(fma((double)o_r, (double)o_r, (double)o_i * (double)o_i))
                                          : hypot((double)o_r, (double)o_i);
      st0 += m0 * m0;
      st1 += (m1 - m0) * (m1 - m0);
      st3 += m1;
    }
  }
  Real* dst = PROX ? s_out : a.gout;
  if (full) {
#pragma unroll
    for (int u = 0; u < NU; ++u)
      reinterpret_cast<U16*>(dst + 2 * n0)[u] = *reinterpret_cast<const U16*>(io + u * (16 / sizeof(Real)));
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (!(x0 + v < g.nx && y < g.ny && z < g.nzs)) continue;
      dst[2 * (n0 + v)] = io[2 * v];
      dst[2 * (n0 + v) + 1] = io[2 * v + 1];
    }
  }
  if (PROX) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st0 += __shfl_xor_sync(FULL, st0, o);
      st1 += __shfl_xor_sync(FULL, st1, o);
      st3 += __shfl_xor_sync(FULL, st3, o);
    }
    if (L == 0) {
      a.stat_part[(size_t)tile * 4 + 0] = st0;
      a.stat_part[(size_t)tile * 4 + 1] = st1;
      a.stat_part[(size_t)tile * 4 + 2] = 0;
      a.stat_part[(size_t)tile * 4 + 3] = st3;
    }
  }
}

// One adjoint warp unit (tile, channel chunk) of the flat kernel: the body of adj_kernel, also run by the
// persistent SPGM loop (spgm_loop_kernel). wbase: this warp's shared-memory region.
template <typename Real, bool PROX, bool EXACT, bool LOOP = false>
__device__ __forceinline__ void adj_unit(const AdjArgs<Real>& a, int unit, unsigned char* wbase, int L,
                                         const Real* __restrict__ s_in, Real* __restrict__ s_out,
                                         const ChanRec* __restrict__ crec_loop = nullptr) {
  const Geo& g = a.g;
  int tile, chunk, C;
  unit_map(unit, g.ntiles, a.CH, a.t1, a.CH2, a.order, tile, chunk, C);
  const WarpSmem<Real> ws = carve<Real>(wbase, g.Tg, g.A);
  const int j0 = chunk_bound(a.B, chunk, C, a.order, a.taper);
  const int j1 = chunk_bound(a.B, chunk + 1, C, a.order, a.taper);
  // Start-up loads that do not depend on the predecessor kernel are issued before griddepcontrol.wait:
  // the D0 row (plan data) and the channel records (written by nf_batch_prepare, whose kernels completed
  // before the residual kernel, our predecessor, released us). The residual records w come after the wait.
  ChanRec nxt;
  R2<Real> nxtw;
  prefetch_first<Real>(LOOP ? crec_loop : a.crec, nullptr, j0, j1, L, nxt, nxtw);
  for (int i = L; i < g.A; i += 32) ws.d0[i] = a.D0[(size_t)tile * g.A + i];
  for (int i = L; i < 34; i += 32) ws.rect[i] = make_int2(0, -1);
  pdl_wait();
  if (j0 + L < j1) nxtw = a.wrec[j0 + L];
  __syncwarp();
  const Real* tabt = a.tab + (size_t)tile * g.A * TABW;
  const Real* tsl = ws.tside + L * (16 / (int)sizeof(Real));

  QV<Real> gr, gi, hr, hi, dR, iR;
  zero(gr);
  zero(gi);
  zero(hr);
  zero(hi);
  zero(dR);
  zero(iR);
  int cur_tg = -1, pf_r = -1, carry = -1, rslot = 0;

  for (int jb = j0; jb < j1; jb += 32) {
    const int nb = min(32, j1 - jb);
    const unsigned starts = build_records<Real, EXACT>(g, ws, LOOP ? crec_loop : a.crec, a.wrec, jb, nb, j1, L, carry, nxt,
                                                             nxtw);
    int c = 0;
    while (c < nb) {
      const int key = ws.rect[c].y;
      const int e = key >> 24;
      if ((starts >> c) & 1u) {  // a new (rx, tx-group) run begins at c
        const int rr = key & 0x7fff, tg = (key >> 15) & 0x1ff;
        if (tg != cur_tg) {
          load_tgroup_async<Real>(g, tabt, ws.tside, tg, L);
          cur_tg = tg;
        }
        flush(iR, hr, hi, gr, gi);
        rx_run_rows<Real>(g, tabt, ws, rr, pf_r, rslot, L, dR, iR);
      }
      // software pipeline: channel c+1's record loads while c computes
      R4<Real> q = ws.rec[c];
      int off = low2(q.y) * TABW;
#pragma unroll UNROLL
      for (; c < e; ++c) {
        const R4<Real> qn = ws.rec[c + 1];
        const int offn = low2(qn.y) * TABW;
        const QV<Real> dT = ldv(tsl + off), iT = ldv(tsl + off + TILE);
        QV<Real> cs, sn;
        phasorv<EXACT>(q.x, q.y, dT, dR, cs, sn);
        adj_acc(iT, cs, sn, q.z, q.w, hr, hi);
        q = qn;
        off = offn;
      }
    }
    __syncwarp();
  }
  flush(iR, hr, hi, gr, gi);
  stage_wait();

  adj_epilogue<Real, PROX, LOOP>(a, tile, chunk, C, L, gr, gi, s_in, s_out);
}

template <typename Real, bool PROX, bool EXACT>
__global__ void __launch_bounds__(ADJ_WARPS * 32, NFGPU_MINB_ADJ) adj_kernel(AdjArgs<Real> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int unit = blockIdx.x * ADJ_WARPS + w;
  if (unit >= a.t1 * a.CH + (a.g.ntiles - a.t1) * a.CH2) return;  // warps are independent: no block barriers
  adj_unit<Real, PROX, EXACT>(a, unit, smem_raw + (size_t)w * warp_smem_bytes<Real>(a.g.Tg, a.g.A), L, a.s_in,
                              a.s_out);
}

// stats = {Σ_tile part[.][0], Σ part[.][1], ½ Σ_block dpart, Σ part[.][3]} in a fixed order
__global__ void __launch_bounds__(256) stats_reduce_kernel(const double* __restrict__ part, int n,
                                                           const double* __restrict__ dpart, int nd,
                                                           double* __restrict__ out) {
  pdl_wait_and_release();
  __shared__ double sh[4][256];
  double acc[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < n; i += 256) {
    acc[0] += part[(size_t)i * 4 + 0];
    acc[1] += part[(size_t)i * 4 + 1];
    acc[3] += part[(size_t)i * 4 + 3];
  }
  for (int i = threadIdx.x; i < nd; i += 256) acc[2] += dpart[i];
#pragma unroll
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 4) out[threadIdx.x] = threadIdx.x == 2 ? 0.5 * sh[2][0] : sh[threadIdx.x][0];
}

// ------------------------------------------------------------------ forward
template <typename Real>
struct FwdArgs {
  Geo g;
  const Real* __restrict__ tab;
  const double* __restrict__ D0;
  const ChanRec* __restrict__ crec;
  const Real* __restrict__ s;  // complex, slab-local flat order
  int w0, w1;                  // sorted positions of this launch window
  int Q;                       // channel splits per tile
  int order;                   // unit order, as AdjArgs::order
  int t1, Q2;                  // tile-major tail, as AdjArgs::t1/CH2
  float taper;                 // as AdjArgs::taper
  Real* __restrict__ part;     // [gridDim.x][w1-w0] complex
};

template <typename Real>
__host__ __device__ constexpr size_t fwd_warp_bytes(int Tg, int A) {
  return warp_smem_bytes<Real>(Tg, A, 1) + (size_t)TBR * 33 * sizeof(R2<Real>);
}

// Sum of one element from each of the four (c64) / eight (c128) shared loads of ldv(dR), ldv(iR):
// consuming it makes an instruction wait until every load of the slot has returned its data.
__device__ __forceinline__ float slot_guard(const FV& dR, const FV& iR) {
  return (dR.p[0].x + dR.p[NP / 2].x) + (iR.p[0].x + iR.p[NP / 2].x);
}
__device__ __forceinline__ double slot_guard(const DV& dR, const DV& iR) {
  double t = 0;
#pragma unroll
  for (int i = 0; i < V; i += 2) t += dR.v[i] + iR.v[i];
  return t;
}

// Forward variant with ONE staging slot: read the prefetched rows of receiver rr into registers,
// then start the prefetch of the next receiver into the same slot. The prefetch is predicated on
// a value computed from every load of the slot (always true: table entries are finite), so it
// cannot be issued before those loads have completed (no write-after-read race on the slot).
template <typename Real>
__device__ __forceinline__ void rx_run_rows_1slot(const Geo& g, const Real* __restrict__ tabt,
                                                  const WarpSmem<Real>& ws, int rr, int& pf_r, int L, QV<Real>& dR,
                                                  QV<Real>& iR) {
  if (rr != pf_r) {  // not prefetched: drain any stale prefetch into the slot, then stage rr
    stage_wait();
    stage_rx<Real>(g, tabt, rr, ws.rslot, L);
  }
  stage_wait();
  __syncwarp();  // a tx-group copy issued at this run start is complete for every lane
  const Real* src = ws.rslot + L * (16 / (int)sizeof(Real));
  dR = ldv(src);
  iR = ldv(src + TILE);
  pf_r = rr + 1 < g.R ? rr + 1 : 0;
  const Real guard = slot_guard(dR, iR);
  if (guard == guard) stage_rx<Real>(g, tabt, pf_r, ws.rslot, L);
}

// Forward: a warp owns (tile, channel chunk) like the adjoint. Per channel, each lane forms
// the sum over its V voxels. Every 16 channels, a transpose through smem reduces over the
// 32 lanes in a fixed order, and the tile's per-channel sum goes to part[tile][j].
// With tile-major units (large tables), chunks of one tile are adjacent units, so they run
// together and share the tile's table rows in L2.
// One forward warp unit (tile, channel chunk): the body of fwd_kernel, also run by spgm_loop_kernel.
// LOOP = false (fwd_kernel): the iterate is a.s and the warp's region follows fwd_warp_bytes, as written inline
// in the kernel (keeps its code generation); LOOP = true: the iterate sv_loop and the region wbase_loop.
template <typename Real, bool EXACT, bool LOOP = false>
__device__ __forceinline__ void fwd_unit(const FwdArgs<Real>& a, int unit, unsigned char* smem_base, int w, int L,
                                         const Real* __restrict__ sv_loop = nullptr,
                                         const ChanRec* __restrict__ crec_loop = nullptr) {
  const Geo& g = a.g;
  int tile, chunk, C;
  unit_map(unit, g.ntiles, a.Q, a.t1, a.Q2, a.order, tile, chunk, C);
  const ChanRec* __restrict__ crec = LOOP ? crec_loop : a.crec;
  unsigned char* wbase = LOOP ? smem_base : smem_base + (size_t)w * fwd_warp_bytes<Real>(g.Tg, g.A);
  const Real* __restrict__ sv = LOOP ? sv_loop : a.s;
  const WarpSmem<Real> ws = carve<Real>(wbase, g.Tg, g.A, 1);
  R2<Real>* tb = reinterpret_cast<R2<Real>*>(wbase + warp_smem_bytes<Real>(g.Tg, g.A, 1));  // [TBR][33]

  // Start-up loads: the lane's s values and the D0 row do not depend on the predecessor kernel (the
  // last of nf_batch_prepare's kernels, which waited for everything before it), so they are issued
  // before griddepcontrol.wait; the channel records it writes come after.
  const int span = a.w1 - a.w0;
  const int c0 = a.w0 + chunk_bound(span, chunk, C, a.order, a.taper);
  const int c1 = a.w0 + chunk_bound(span, chunk + 1, C, a.order, a.taper);
  R2<Real>* out = reinterpret_cast<R2<Real>*>(a.part) + (size_t)tile * span - a.w0;
  ChanRec nxt;
  R2<Real> nxtw;
  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(tx, ty, tz, L, x0, y, z);
  Real srv[V], siv[V];
  {  // the lane's V voxels (consecutive in x): 16-byte vector loads when all are inside and aligned
    using U16 = typename std::conditional<std::is_same<Real, float>::value, float4, double2>::type;
    constexpr int NU = 2 * V * (int)sizeof(Real) / 16, PU = 16 / (int)sizeof(Real);
    const size_t n0 = ((size_t)z * g.ny + y) * g.nx + x0;
    if (x0 + V <= g.nx && y < g.ny && z < g.nzs && (sizeof(Real) == 8 || (g.nx & 1) == 0)) {
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const U16 w = LOOP ? __ldcg(reinterpret_cast<const U16*>(sv + 2 * n0) + u)
                           : reinterpret_cast<const U16*>(sv + 2 * n0)[u];
        const Real* t = reinterpret_cast<const Real*>(&w);
#pragma unroll
        for (int k = 0; k < PU; k += 2) {
          srv[(u * PU + k) >> 1] = t[k];
          siv[(u * PU + k) >> 1] = t[k + 1];
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool ok = x0 + v < g.nx && y < g.ny && z < g.nzs;
        srv[v] = ok ? (LOOP ? __ldcg(sv + 2 * (n0 + v)) : sv[2 * (n0 + v)]) : Real(0);
        siv[v] = ok ? (LOOP ? __ldcg(sv + 2 * (n0 + v) + 1) : sv[2 * (n0 + v) + 1]) : Real(0);
      }
    }
  }
  for (int i = L; i < g.A; i += 32) ws.d0[i] = a.D0[(size_t)tile * g.A + i];
  for (int i = L; i < 34; i += 32) ws.rect[i] = make_int2(0, -1);
  pdl_wait();
  prefetch_first<Real>(crec, nullptr, c0, c1, L, nxt, nxtw);
  const Real* tabt = a.tab + (size_t)tile * g.A * TABW;
  const Real* tsl = ws.tside + L * (16 / (int)sizeof(Real));
  const QV<Real> sr = make_v(srv), si = make_v(siv);
  int cur_tg = -1, pf_r = -1, carry = -1;
  if (c0 < c1) {  // stage the first run's tx group and rx rows as soon as the first record is in
    const int pk0 = __shfl_sync(FULL, nxt.pk, 0);
    cur_tg = tx_group(g, pk_t(pk0));
    pf_r = pk_r(pk0);
    load_tgroup_async<Real>(g, tabt, ws.tside, cur_tg, L);
    stage_rx<Real>(g, tabt, pf_r, ws.rslot, L);
  }
  __syncwarp();

  QV<Real> dR, iR, shr, shi, nshr;
  zero(dR);
  zero(iR);
  zero(shr);
  zero(shi);
  zero(nshr);
  R2<Real>* outl = out + L;
  for (int jb = c0; jb < c1; jb += 32) {
    const int nb = min(32, c1 - jb);
    const unsigned starts =
        build_records<Real, EXACT>(g, ws, crec, nullptr, jb, nb, c1, L, carry, nxt, nxtw);
    // sub-batches of TBR channels share one [TBR][33] transpose buffer
    for (int h0 = 0; h0 < nb; h0 += TBR) {
      const int h1 = min(nb, h0 + TBR);
      int c = h0;
      while (c < h1) {
        const int key = ws.rect[c].y;
        const int e = min(key >> 24, h1);
        if ((starts >> c) & 1u) {  // a new (rx, tx-group) run begins at c
          const int rr = key & 0x7fff, tg = (key >> 15) & 0x1ff;
          if (tg != cur_tg) {
            load_tgroup_async<Real>(g, tabt, ws.tside, tg, L);
            cur_tg = tg;
          }
          rx_run_rows_1slot<Real>(g, tabt, ws, rr, pf_r, L, dR, iR);
          scale_s(iR, sr, si, shr, shi, nshr);
        }
        // two channels per iteration, both results stored after both are computed, so the
        // compiler can overlap their dependency chains (a store in between would be a barrier)
        for (; c + 1 < e; c += 2) {
          const R4<Real> q0 = ws.rec[c], q1 = ws.rec[c + 1];
          const int o0 = bits_int(q0.z), o1 = bits_int(q1.z);
          const QV<Real> dT0 = ldv(tsl + o0), iT0 = ldv(tsl + o0 + TILE);
          const QV<Real> dT1 = ldv(tsl + o1), iT1 = ldv(tsl + o1 + TILE);
          QV<Real> cs0, sn0, cs1, sn1;
          phasorv<EXACT, NFGPU_FWD_CIS>(q0.x, q0.y, dT0, dR, cs0, sn0);
          phasorv<EXACT, NFGPU_FWD_CIS>(q1.x, q1.y, dT1, dR, cs1, sn1);
          const R2<Real> p0 = fwd_part(iT0, cs0, sn0, shr, shi, nshr);
          const R2<Real> p1 = fwd_part(iT1, cs1, sn1, shr, shi, nshr);
          tb[(c - h0) * 33 + L] = p0;
          tb[(c + 1 - h0) * 33 + L] = p1;
        }
        if (c < e) {
          const R4<Real> q = ws.rec[c];
          const int off = bits_int(q.z);
          const QV<Real> dT = ldv(tsl + off), iT = ldv(tsl + off + TILE);
          QV<Real> cs, sn;
          phasorv<EXACT, NFGPU_FWD_CIS>(q.x, q.y, dT, dR, cs, sn);
          tb[(c - h0) * 33 + L] = fwd_part(iT, cs, sn, shr, shi, nshr);
          ++c;
        }
      }
      __syncwarp();
      // transpose-reduce: 32/TBR lanes per row each sum a 32/(32/TBR) slice of row L % TBR,
      // then combine with shuffles (fixed order)
      constexpr int PER = 32 / TBR, SL = 32 / PER;
      const int row = L % TBR, part = L / TBR;
      R2<Real> S;
      S.x = 0;
      S.y = 0;
#pragma unroll 8
      for (int l = 0; l < SL; ++l) {
        const R2<Real> t = tb[row * 33 + part * SL + l];
        if constexpr (std::is_same<Real, float>::value) {
          S = add2(S, t);
        } else {
          S.x += t.x;
          S.y += t.y;
        }
      }
#pragma unroll
      for (int o = 16; o >= TBR; o >>= 1) {
        S.x += __shfl_down_sync(FULL, S.x, o);
        S.y += __shfl_down_sync(FULL, S.y, o);
      }
      if (L < h1 - h0) outl[jb + h0] = S;
      __syncwarp();
    }
  }
  stage_wait();
}

// fwd_kernel keeps its own copy of the unit body (the same source as fwd_unit, which the persistent loop runs):
// routing it through fwd_unit changes ptxas's schedule of the kernel and costs 1.8% on Large (2.437 -> 2.480 ms)
template <typename Real, bool EXACT>
__global__ void __launch_bounds__(FWD_WARPS * 32, NFGPU_MINB_FWD) fwd_kernel(FwdArgs<Real> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& g = a.g;
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int unit = blockIdx.x * FWD_WARPS + w;
  if (unit >= a.t1 * a.Q + (g.ntiles - a.t1) * a.Q2) return;  // warps are independent: no block barriers
  int tile, chunk, C;
  unit_map(unit, g.ntiles, a.Q, a.t1, a.Q2, a.order, tile, chunk, C);
  unsigned char* wbase = smem_raw + (size_t)w * fwd_warp_bytes<Real>(g.Tg, g.A);
  const WarpSmem<Real> ws = carve<Real>(wbase, g.Tg, g.A, 1);
  R2<Real>* tb = reinterpret_cast<R2<Real>*>(wbase + warp_smem_bytes<Real>(g.Tg, g.A, 1));  // [TBR][33]

  // Start-up loads: the lane's s values and the D0 row do not depend on the predecessor kernel (the
  // last of nf_batch_prepare's kernels, which waited for everything before it), so they are issued
  // before griddepcontrol.wait; the channel records it writes come after.
  const int span = a.w1 - a.w0;
  const int c0 = a.w0 + chunk_bound(span, chunk, C, a.order, a.taper);
  const int c1 = a.w0 + chunk_bound(span, chunk + 1, C, a.order, a.taper);
  R2<Real>* out = reinterpret_cast<R2<Real>*>(a.part) + (size_t)tile * span - a.w0;
  ChanRec nxt;
  R2<Real> nxtw;
  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(tx, ty, tz, L, x0, y, z);
  Real srv[V], siv[V];
  {  // the lane's V voxels (consecutive in x): 16-byte vector loads when all are inside and aligned
    using U16 = typename std::conditional<std::is_same<Real, float>::value, float4, double2>::type;
    constexpr int NU = 2 * V * (int)sizeof(Real) / 16, PU = 16 / (int)sizeof(Real);
    const size_t n0 = ((size_t)z * g.ny + y) * g.nx + x0;
    if (x0 + V <= g.nx && y < g.ny && z < g.nzs && (sizeof(Real) == 8 || (g.nx & 1) == 0)) {
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const U16 w = reinterpret_cast<const U16*>(a.s + 2 * n0)[u];
        const Real* t = reinterpret_cast<const Real*>(&w);
#pragma unroll
        for (int k = 0; k < PU; k += 2) {
          srv[(u * PU + k) >> 1] = t[k];
          siv[(u * PU + k) >> 1] = t[k + 1];
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool ok = x0 + v < g.nx && y < g.ny && z < g.nzs;
        srv[v] = ok ? a.s[2 * (n0 + v)] : Real(0);
        siv[v] = ok ? a.s[2 * (n0 + v) + 1] : Real(0);
      }
    }
  }
  for (int i = L; i < g.A; i += 32) ws.d0[i] = a.D0[(size_t)tile * g.A + i];
  for (int i = L; i < 34; i += 32) ws.rect[i] = make_int2(0, -1);
  pdl_wait();
  prefetch_first<Real>(a.crec, nullptr, c0, c1, L, nxt, nxtw);
  const Real* tabt = a.tab + (size_t)tile * g.A * TABW;
  const Real* tsl = ws.tside + L * (16 / (int)sizeof(Real));
  const QV<Real> sr = make_v(srv), si = make_v(siv);
  int cur_tg = -1, pf_r = -1, carry = -1;
  if (c0 < c1) {  // stage the first run's tx group and rx rows as soon as the first record is in
    const int pk0 = __shfl_sync(FULL, nxt.pk, 0);
    cur_tg = tx_group(g, pk_t(pk0));
    pf_r = pk_r(pk0);
    load_tgroup_async<Real>(g, tabt, ws.tside, cur_tg, L);
    stage_rx<Real>(g, tabt, pf_r, ws.rslot, L);
  }
  __syncwarp();

  QV<Real> dR, iR, shr, shi, nshr;
  zero(dR);
  zero(iR);
  zero(shr);
  zero(shi);
  zero(nshr);
  R2<Real>* outl = out + L;
  for (int jb = c0; jb < c1; jb += 32) {
    const int nb = min(32, c1 - jb);
    const unsigned starts =
        build_records<Real, EXACT>(g, ws, a.crec, nullptr, jb, nb, c1, L, carry, nxt, nxtw);
    // sub-batches of TBR channels share one [TBR][33] transpose buffer
    for (int h0 = 0; h0 < nb; h0 += TBR) {
      const int h1 = min(nb, h0 + TBR);
      int c = h0;
      while (c < h1) {
        const int key = ws.rect[c].y;
        const int e = min(key >> 24, h1);
        if ((starts >> c) & 1u) {  // a new (rx, tx-group) run begins at c
          const int rr = key & 0x7fff, tg = (key >> 15) & 0x1ff;
          if (tg != cur_tg) {
            load_tgroup_async<Real>(g, tabt, ws.tside, tg, L);
            cur_tg = tg;
          }
          rx_run_rows_1slot<Real>(g, tabt, ws, rr, pf_r, L, dR, iR);
          scale_s(iR, sr, si, shr, shi, nshr);
        }
        // two channels per iteration, both results stored after both are computed, so the
        // compiler can overlap their dependency chains (a store in between would be a barrier)
        for (; c + 1 < e; c += 2) {
          const R4<Real> q0 = ws.rec[c], q1 = ws.rec[c + 1];
          const int o0 = bits_int(q0.z), o1 = bits_int(q1.z);
          const QV<Real> dT0 = ldv(tsl + o0), iT0 = ldv(tsl + o0 + TILE);
          const QV<Real> dT1 = ldv(tsl + o1), iT1 = ldv(tsl + o1 + TILE);
          QV<Real> cs0, sn0, cs1, sn1;
          phasorv<EXACT, NFGPU_FWD_CIS>(q0.x, q0.y, dT0, dR, cs0, sn0);
          phasorv<EXACT, NFGPU_FWD_CIS>(q1.x, q1.y, dT1, dR, cs1, sn1);
          const R2<Real> p0 = fwd_part(iT0, cs0, sn0, shr, shi, nshr);
          const R2<Real> p1 = fwd_part(iT1, cs1, sn1, shr, shi, nshr);
          tb[(c - h0) * 33 + L] = p0;
          tb[(c + 1 - h0) * 33 + L] = p1;
        }
        if (c < e) {
          const R4<Real> q = ws.rec[c];
          const int off = bits_int(q.z);
          const QV<Real> dT = ldv(tsl + off), iT = ldv(tsl + off + TILE);
          QV<Real> cs, sn;
          phasorv<EXACT, NFGPU_FWD_CIS>(q.x, q.y, dT, dR, cs, sn);
          tb[(c - h0) * 33 + L] = fwd_part(iT, cs, sn, shr, shi, nshr);
          ++c;
        }
      }
      __syncwarp();
      // transpose-reduce: 32/TBR lanes per row each sum a 32/(32/TBR) slice of row L % TBR,
      // then combine with shuffles (fixed order)
      constexpr int PER = 32 / TBR, SL = 32 / PER;
      const int row = L % TBR, part = L / TBR;
      R2<Real> S;
      S.x = 0;
      S.y = 0;
#pragma unroll 8
      for (int l = 0; l < SL; ++l) {
        const R2<Real> t = tb[row * 33 + part * SL + l];
        if constexpr (std::is_same<Real, float>::value) {
          S = add2(S, t);
        } else {
          S.x += t.x;
          S.y += t.y;
        }
      }
#pragma unroll
      for (int o = 16; o >= TBR; o >>= 1) {
        S.x += __shfl_down_sync(FULL, S.x, o);
        S.y += __shfl_down_sync(FULL, S.y, o);
      }
      if (L < h1 - h0) outl[jb + h0] = S;
      __syncwarp();
    }
  }
  stage_wait();
}

// ------------------------------------------------------------------ structured (Cartesian) batches
//
// SURVEY.md §8(f) #2. A structured minibatch (solver.py:206-225, the reference's own sampler) is
// Fs × Ts × Rs in lexicographic (f, t, r) order. Then
//     A[(f,t,r), n] = p_f/(4π) · U_ft(n) · V_fr(n),   U = e^{-j2π(f/c) d_T}/d_T,  V = e^{-j2π(f/c) d_R}/d_R
// so per frequency a voxel needs n_t + n_r phasors instead of n_t·n_r. The contraction over the
// batch becomes complex multiply-adds on the FMA pipe: the adjoint computes
// Σ_t conj(U_ft)·Σ_r conj(V_fr)·w_ftr, and the forward computes Σ_n U_ft·(V_fr·s) per (t, r).
// A block of SW warps owns (tile, chunk of (f, t) rows). Per frequency, the warps jointly stage
// the rx factors of RBS receivers in shared memory (each warp computes every SW-th row). Each
// warp then takes its own blocks of TB transmitters, held in registers, so one shared-memory
// load of an rx factor feeds TB complex multiply-adds. The tx table rows of the next
// transmitter block are prefetched per lane with cp.async while the contraction runs.

constexpr int SW = 4;  // warps per structured block
template <typename Real>
struct SCfg;
template <>
struct SCfg<float> {
  static constexpr int TB = 4, RBA = 16, RBF = 12;
};
template <>
struct SCfg<double> {
  static constexpr int TB = 2, RBA = 8, RBF = 6;
};

// block shared-memory layout: stage | s (forward) | D0 row | SW × per-warp area
template <typename Real, bool FWD>
struct SLayout {
  static constexpr int TB = SCfg<Real>::TB;
  static constexpr int RBS = FWD ? SCfg<Real>::RBF : SCfg<Real>::RBA;
  static constexpr size_t stage = (size_t)RBS * 2 * TILE * sizeof(Real);
  static constexpr size_t sv = FWD ? (size_t)2 * TILE * sizeof(Real) : 0;
  static constexpr size_t trow = (size_t)TB * TABW * sizeof(Real);
  static constexpr size_t wsm = FWD ? 0 : (size_t)RBS * TB * sizeof(R2<Real>);
  static constexpr size_t tbuf = FWD ? (size_t)TBR * 33 * sizeof(R2<Real>) + 16 * sizeof(int) : 0;
  static constexpr size_t warp = trow + wsm + ((tbuf + 15) & ~(size_t)15);
  __host__ __device__ static constexpr size_t bytes(int A) {
    return stage + sv + (size_t)d0_slots(A) * sizeof(double) + SW * warp;
  }
};

struct StructArgs {
  const int* __restrict__ fs;
  const int* __restrict__ ts;
  const int* __restrict__ rs;
  int nf, nt, nr;
};

// copy antenna a's table rows (δ and 1/d blocks) for this lane's voxels into slot; each lane
// copies and later reads back only its own quads (see stage_rx)
template <typename Real>
__device__ __forceinline__ void stage_row(const Real* __restrict__ tabt, int a, Real* slot, int L) {
  constexpr int QD = 16 / (int)sizeof(Real);
  const Real* src = tabt + (size_t)a * TABW + L * QD;
  Real* dst = slot + L * QD;
  constexpr int n16 = V / QD;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < n16; ++i) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + h * TILE + i * 32 * QD);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + h * TILE + i * 32 * QD)
                   : "memory");
    }
}
__device__ __forceinline__ void stage_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

__device__ __forceinline__ void stv(float* p, const FV& q) {
#pragma unroll
  for (int i = 0; i < NP / 2; ++i)
    *reinterpret_cast<float4*>(p + i * 128) = make_float4(q.p[2 * i].x, q.p[2 * i].y, q.p[2 * i + 1].x, q.p[2 * i + 1].y);
}
__device__ __forceinline__ void stv(double* p, const DV& q) {
#pragma unroll
  for (int i = 0; i < V / 2; ++i) *reinterpret_cast<double2*>(p + i * 64) = make_double2(q.v[2 * i], q.v[2 * i + 1]);
}

// One-sided phase parameters for antenna a at frequency f on this tile: slope k and offset b,
// in revolutions (exact path, c128) or radians (fast c64 path), x = b + k·δ.
template <typename Real, bool EXACT>
__device__ __forceinline__ void side_params(double kd, double d0, Real& k, Real& b) {
  const double x = kd * d0;
  const double fr = x - rint(x);
  if (std::is_same<Real, float>::value && !EXACT) {
    k = (Real)(2.0 * PI * kd);
    b = (Real)(2.0 * PI * fr);
  } else {
    k = (Real)kd;
    b = (Real)fr;
  }
}

// amplitude-weighted one-sided phasor: (re, im) = amp·(cos x, sgn·sin x)
template <bool EXACT>
__device__ __forceinline__ void side_phasor(float k, float b, const FV& d, const FV& amp, float sgn, FV& re, FV& im) {
  const float2 M2 = bc(12582912.0f);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const float2 x = fma2(bc(k), d.p[i], bc(b));
    float2 r = x;
    if (EXACT) r = mul2(sub2(x, sub2(add2(x, M2), M2)), bc(6.28318530717958647692f));
    float2 c, sn;
    __sincosf(r.x, &sn.x, &c.x);
    __sincosf(r.y, &sn.y, &c.y);
    re.p[i] = mul2(amp.p[i], c);
    im.p[i] = mul2(amp.p[i], mul2(sn, bc(sgn)));
  }
}
template <bool EXACT>
__device__ __forceinline__ void side_phasor(double k, double b, const DV& d, const DV& amp, double sgn, DV& re, DV& im) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double x = fma(k, d.v[v], b);
    double c, sn;
    cis_rev(x - rint(x), sn, c);
    re.v[v] = amp.v[v] * c;
    im.v[v] = amp.v[v] * sgn * sn;
  }
}

// z += v · w  (lane vector × complex scalar)
__device__ __forceinline__ void cmac_s(const FV& vr, const FV& vi, float wr, float wi, FV& zr, FV& zi) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    zr.p[i] = fma2(vi.p[i], bc(-wi), fma2(vr.p[i], bc(wr), zr.p[i]));
    zi.p[i] = fma2(vi.p[i], bc(wr), fma2(vr.p[i], bc(wi), zi.p[i]));
  }
}
__device__ __forceinline__ void cmac_s(const DV& vr, const DV& vi, double wr, double wi, DV& zr, DV& zi) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    zr.v[v] = fma(-vi.v[v], wi, fma(vr.v[v], wr, zr.v[v]));
    zi.v[v] = fma(vi.v[v], wr, fma(vr.v[v], wi, zi.v[v]));
  }
}
// z += u · x  (elementwise complex lane vectors)
__device__ __forceinline__ void cmac_v(const FV& ur, const FV& ui, const FV& xr, const FV& xi, FV& zr, FV& zi) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    zr.p[i] = fma2(ui.p[i], make_float2(-xi.p[i].x, -xi.p[i].y), fma2(ur.p[i], xr.p[i], zr.p[i]));
    zi.p[i] = fma2(ui.p[i], xr.p[i], fma2(ur.p[i], xi.p[i], zi.p[i]));
  }
}
__device__ __forceinline__ void cmac_v(const DV& ur, const DV& ui, const DV& xr, const DV& xi, DV& zr, DV& zi) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    zr.v[v] = fma(-ui.v[v], xi.v[v], fma(ur.v[v], xr.v[v], zr.v[v]));
    zi.v[v] = fma(ui.v[v], xr.v[v], fma(ur.v[v], xi.v[v], zi.v[v]));
  }
}
// Σ_v u·w over the lane's voxels (complex); two accumulator chains per component
__device__ __forceinline__ float2 cdot(const FV& ur, const FV& ui, const FV& wr, const FV& wi) {
  float2 pr0 = make_float2(0.f, 0.f), pi0 = pr0, pr1 = pr0, pi1 = pr0;
#pragma unroll
  for (int i = 0; i < NP; i += 2) {
    pr0 = fma2(ui.p[i], make_float2(-wi.p[i].x, -wi.p[i].y), fma2(ur.p[i], wr.p[i], pr0));
    pi0 = fma2(ui.p[i], wr.p[i], fma2(ur.p[i], wi.p[i], pi0));
    pr1 = fma2(ui.p[i + 1], make_float2(-wi.p[i + 1].x, -wi.p[i + 1].y), fma2(ur.p[i + 1], wr.p[i + 1], pr1));
    pi1 = fma2(ui.p[i + 1], wr.p[i + 1], fma2(ur.p[i + 1], wi.p[i + 1], pi1));
  }
  const float2 pr = add2(pr0, pr1), pi = add2(pi0, pi1);
  return make_float2(pr.x + pr.y, pi.x + pi.y);
}
__device__ __forceinline__ double2 cdot(const DV& ur, const DV& ui, const DV& wr, const DV& wi) {
  double pr0 = 0, pi0 = 0, pr1 = 0, pi1 = 0;
#pragma unroll
  for (int v = 0; v < V; v += 2) {
    pr0 = fma(-ui.v[v], wi.v[v], fma(ur.v[v], wr.v[v], pr0));
    pi0 = fma(ui.v[v], wr.v[v], fma(ur.v[v], wi.v[v], pi0));
    pr1 = fma(-ui.v[v + 1], wi.v[v + 1], fma(ur.v[v + 1], wr.v[v + 1], pr1));
    pi1 = fma(ui.v[v + 1], wr.v[v + 1], fma(ur.v[v + 1], wi.v[v + 1], pi1));
  }
  return make_double2(pr0 + pr1, pi0 + pi1);
}

// Rows u = fi·nt + ti of a structured batch; a block owns the row range [u0, u1), which
// covers transmitters [ta, tb) of frequency fi.
__device__ __forceinline__ void row_span(const StructArgs& sa, int u0, int u1, int fi, int& ta, int& tb) {
  ta = max(u0, fi * sa.nt) - fi * sa.nt;
  tb = min(u1, (fi + 1) * sa.nt) - fi * sa.nt;
}

#ifndef NFGPU_MINB_STRUCT
#define NFGPU_MINB_STRUCT 3
#endif

// Structured adjoint (+prox): g = Σ_f Σ_t conj(U_ft)·Σ_r conj(V_fr)·w_ftr. Block = (tile, row chunk).
template <typename Real, bool PROX, bool EXACT>
__global__ void __launch_bounds__(SW * 32, NFGPU_MINB_STRUCT) adj_struct_kernel(AdjArgs<Real> a, StructArgs sa,
                                                                              const double* __restrict__ kd) {
  using LY = SLayout<Real, false>;
  constexpr int TB = LY::TB, RBS = LY::RBS;
  constexpr int QD = 16 / (int)sizeof(Real);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& g = a.g;
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int tile = blockIdx.x / a.CH, chunk = blockIdx.x - tile * a.CH;
  Real* stage = reinterpret_cast<Real*>(smem_raw);
  double* d0 = reinterpret_cast<double*>(smem_raw + LY::stage);
  unsigned char* wb = smem_raw + LY::stage + (size_t)d0_slots(g.A) * sizeof(double) + (size_t)w * LY::warp;
  Real* trow = reinterpret_cast<Real*>(wb);
  R2<Real>* wsm = reinterpret_cast<R2<Real>*>(wb + LY::trow);
  for (int i = threadIdx.x; i < g.A; i += SW * 32) d0[i] = a.D0[(size_t)tile * g.A + i];
  __syncthreads();
  const Real* tabt = a.tab + (size_t)tile * g.A * TABW;
  Real* stl = stage + L * QD;
  const Real* trl = trow + L * QD;
  const int rows = sa.nf * sa.nt;
  const int u0 = (int)(((long long)rows * chunk) / a.CH), u1 = (int)(((long long)rows * (chunk + 1)) / a.CH);

  QV<Real> gr, gi;
  zero(gr);
  zero(gi);
  int ld_t0 = -1, ld_tc = 0;  // transmitter block whose rows are in trow
  for (int fi = u0 / sa.nt; fi * sa.nt < u1; ++fi) {
    int ta, tb;
    row_span(sa, u0, u1, fi, ta, tb);
    const double kf = kd[sa.fs[fi]];
    for (int r0 = 0; r0 < sa.nr; r0 += RBS) {
      const int nrb = min(RBS, sa.nr - r0);
      for (int q = w; q < nrb; q += SW) {  // conj(V_fr) rows, shared by the block
        const int ant = g.T + sa.rs[r0 + q];
        const Real* row = tabt + (size_t)ant * TABW + L * QD;
        Real k, b;
        side_params<Real, EXACT>(kf, d0[ant], k, b);
        QV<Real> re, im;
        side_phasor<EXACT>(k, b, ldv(row), ldv(row + TILE), Real(1), re, im);
        stv(stl + (size_t)q * 2 * TILE, re);
        stv(stl + (size_t)q * 2 * TILE + TILE, im);
      }
      __syncthreads();
      for (int t0 = ta + w * TB; t0 < tb; t0 += SW * TB) {
        const int tc = min(TB, tb - t0);
        if (t0 != ld_t0 || tc > ld_tc) {  // rows arrive while the contraction runs
          for (int k = 0; k < tc; ++k) stage_row<Real>(tabt, sa.ts[t0 + k], trow + (size_t)k * TABW, L);
          stage_commit();
          ld_t0 = t0;
          ld_tc = tc;
        }
        __syncwarp();
        for (int i = L; i < nrb * TB; i += 32) {
          const int q = i / TB, k = i - q * TB;
          R2<Real> v;
          v.x = 0;
          v.y = 0;
          if (k < tc) v = a.wrec[((size_t)fi * sa.nt + t0 + k) * sa.nr + r0 + q];
          wsm[i] = v;
        }
        __syncwarp();
        QV<Real> zr[TB], zi[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          zero(zr[k]);
          zero(zi[k]);
        }
        for (int q = 0; q < nrb; ++q) {
          const QV<Real> vr = ldv(stl + (size_t)q * 2 * TILE), vi = ldv(stl + (size_t)q * 2 * TILE + TILE);
#pragma unroll
          for (int k = 0; k < TB; ++k) {
            const R2<Real> wq = wsm[q * TB + k];
            cmac_s(vr, vi, wq.x, wq.y, zr[k], zi[k]);
          }
        }
        stage_wait();
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          if (k < tc) {
            const int t = sa.ts[t0 + k];
            Real kk, b;
            side_params<Real, EXACT>(kf, d0[t], kk, b);
            QV<Real> ur, ui;
            side_phasor<EXACT>(kk, b, ldv(trl + (size_t)k * TABW), ldv(trl + (size_t)k * TABW + TILE), Real(1), ur,
                               ui);
            cmac_v(ur, ui, zr[k], zi[k], gr, gi);
          }
        }
      }
      __syncthreads();
    }
  }
  // the block's warps each hold a partial over their transmitters: combine in warp order
  Real* cb = stage + (size_t)(w * 32 + L) * (2 * V);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    cb[2 * v] = get(gr, v);
    cb[2 * v + 1] = get(gi, v);
  }
  __syncthreads();
  if (w != 0) return;
  Real Gr[V], Gi[V];
#pragma unroll
  for (int v = 0; v < V; ++v) Gr[v] = Gi[v] = 0;
  for (int ww = 0; ww < SW; ++ww) {
    const Real* q = stage + (size_t)(ww * 32 + L) * (2 * V);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      Gr[v] += q[2 * v];
      Gi[v] += q[2 * v + 1];
    }
  }
  adj_epilogue<Real, PROX>(a, tile, chunk, a.CH, L, make_v(Gr), make_v(Gi), a.s_in, a.s_out);
}

// Structured forward: y_ftr = p_f/(4π) Σ_n U_ft(n)·(V_fr(n) s_n). The block stages W_fr = V_fr·s;
// each warp forms, per transmitter of its block and staged receiver, the lane sums over its
// voxels, then a [TBR][33] transpose reduces over the 32 lanes in a fixed order and writes one
// partial per (tile, channel), which fwd_reduce1/2 finish. The launch window is the row range
// [w0/nr, w1/nr) of whole (f, t) rows.
template <typename Real, bool EXACT>
__global__ void __launch_bounds__(SW * 32, NFGPU_MINB_STRUCT) fwd_struct_kernel(FwdArgs<Real> a, StructArgs sa,
                                                                              const double* __restrict__ kd) {
  using LY = SLayout<Real, true>;
  constexpr int TB = LY::TB, RBS = LY::RBS;
  constexpr int QD = 16 / (int)sizeof(Real);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& g = a.g;
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int tile = blockIdx.x / a.Q, chunk = blockIdx.x - tile * a.Q;
  Real* stage = reinterpret_cast<Real*>(smem_raw);
  Real* sv = reinterpret_cast<Real*>(smem_raw + LY::stage);
  double* d0 = reinterpret_cast<double*>(smem_raw + LY::stage + LY::sv);
  unsigned char* wb = smem_raw + LY::stage + LY::sv + (size_t)d0_slots(g.A) * sizeof(double) + (size_t)w * LY::warp;
  Real* trow = reinterpret_cast<Real*>(wb);
  R2<Real>* tbuf = reinterpret_cast<R2<Real>*>(wb + LY::trow);
  int* jrow = reinterpret_cast<int*>(tbuf + TBR * 33);
  for (int i = threadIdx.x; i < g.A; i += SW * 32) d0[i] = a.D0[(size_t)tile * g.A + i];
  if (w == 0) {  // the tile's s values, in the table's lane layout
    int tx, ty, tz;
    tile_coords(g, tile, tx, ty, tz);
    int x0, y, z;
    lane_voxel(tx, ty, tz, L, x0, y, z);
    Real srv[V], siv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int x = x0 + v;
      const bool ok = x < g.nx && y < g.ny && z < g.nzs;
      const size_t n = ((size_t)z * g.ny + y) * g.nx + x;
      srv[v] = ok ? a.s[2 * n] : Real(0);
      siv[v] = ok ? a.s[2 * n + 1] : Real(0);
    }
    stv(sv + L * QD, make_v(srv));
    stv(sv + TILE + L * QD, make_v(siv));
  }
  __syncthreads();
  const Real* tabt = a.tab + (size_t)tile * g.A * TABW;
  Real* stl = stage + L * QD;
  const Real* trl = trow + L * QD;
  const int span = a.w1 - a.w0;
  R2<Real>* out = reinterpret_cast<R2<Real>*>(a.part) + (size_t)tile * span - a.w0;
  const int ua = a.w0 / sa.nr, nrows = span / sa.nr;
  const int u0 = ua + (int)(((long long)nrows * chunk) / a.Q), u1 = ua + (int)(((long long)nrows * (chunk + 1)) / a.Q);
  int nrow = 0;

  auto flush_rows = [&](int cnt) {
    __syncwarp();
    constexpr int PER = 32 / TBR, SL = 32 / PER;
    const int row = L % TBR, part = L / TBR;
    R2<Real> S;
    S.x = 0;
    S.y = 0;
#pragma unroll
    for (int l = 0; l < SL; ++l) {
      const R2<Real> t = tbuf[row * 33 + part * SL + l];
      S.x += t.x;
      S.y += t.y;
    }
#pragma unroll
    for (int o = 16; o >= TBR; o >>= 1) {
      S.x += __shfl_down_sync(FULL, S.x, o);
      S.y += __shfl_down_sync(FULL, S.y, o);
    }
    if (L < cnt) out[jrow[L]] = S;
    __syncwarp();
  };
  auto load_rows = [&](int t0, int tc) {
    for (int k = 0; k < tc; ++k) stage_row<Real>(tabt, sa.ts[t0 + k], trow + (size_t)k * TABW, L);
    stage_commit();
  };

  int ld_t0 = -1, ld_tc = 0;
  for (int fi = u0 / sa.nt; fi * sa.nt < u1; ++fi) {
    int ta, tb;
    row_span(sa, u0, u1, fi, ta, tb);
    const double kf = kd[sa.fs[fi]];
    for (int r0 = 0; r0 < sa.nr; r0 += RBS) {
      const int nrb = min(RBS, sa.nr - r0);
      const int first = ta + w * TB;
      if (first < tb && (first != ld_t0 || min(TB, tb - first) > ld_tc)) {  // overlaps the staging below
        ld_t0 = first;
        ld_tc = min(TB, tb - first);
        load_rows(ld_t0, ld_tc);
      }
      {
        const QV<Real> sr = ldv(sv + L * QD), si = ldv(sv + TILE + L * QD);
        for (int q = w; q < nrb; q += SW) {  // W_fr = V_fr·s rows, shared by the block
          const int ant = g.T + sa.rs[r0 + q];
          const Real* row = tabt + (size_t)ant * TABW + L * QD;
          Real k, b;
          side_params<Real, EXACT>(kf, d0[ant], k, b);
          QV<Real> vr, vi, wr, wi;
          side_phasor<EXACT>(k, b, ldv(row), ldv(row + TILE), Real(-1), vr, vi);
          zero(wr);
          zero(wi);
          cmac_v(vr, vi, sr, si, wr, wi);
          stv(stl + (size_t)q * 2 * TILE, wr);
          stv(stl + (size_t)q * 2 * TILE + TILE, wi);
        }
      }
      __syncthreads();
      for (int t0 = first; t0 < tb; t0 += SW * TB) {
        const int tc = min(TB, tb - t0);
        stage_wait();
        QV<Real> ur[TB], ui[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          zero(ur[k]);
          zero(ui[k]);
          if (k < tc) {
            const int t = sa.ts[t0 + k];
            Real kk, b;
            side_params<Real, EXACT>(kf, d0[t], kk, b);
            side_phasor<EXACT>(kk, b, ldv(trl + (size_t)k * TABW), ldv(trl + (size_t)k * TABW + TILE), Real(-1),
                               ur[k], ui[k]);
          }
        }
        const int n0 = t0 + SW * TB;
        if (n0 < tb) {  // rows are consumed: prefetch the next block of this warp
          ld_t0 = n0;
          ld_tc = min(TB, tb - n0);
          load_rows(ld_t0, ld_tc);
        }
        const int jb = (fi * sa.nt + t0) * sa.nr + r0;
        for (int q = 0; q < nrb; ++q) {
          const QV<Real> wr = ldv(stl + (size_t)q * 2 * TILE), wi = ldv(stl + (size_t)q * 2 * TILE + TILE);
          R2<Real> pv[TB];  // all TB dot products first (independent chains), then the row stores
#pragma unroll
          for (int k = 0; k < TB; ++k) pv[k] = cdot(ur[k], ui[k], wr, wi);
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if (k < tc) tbuf[(nrow + k) * 33 + L] = pv[k];
          if (L < tc) jrow[nrow + L] = jb + L * sa.nr + q;
          nrow += tc;
          if (nrow > TBR - TB) {
            flush_rows(nrow);
            nrow = 0;
          }
        }
      }
      __syncthreads();
    }
  }
  if (nrow) flush_rows(nrow);
  stage_wait();
}

// ------------------------------------------------------------------ structured adjoint on tcgen05
//
// Per (tile, f) the structured adjoint's contraction is a real GEMM (c64 only):
//   Z[n][2t+c'] = Σ_k A[n][k] · B[2t+c'][k],   k = 2r + c,
//   A[n][2r] + j·A[n][2r+1] = conj(V_fr(n))  (generated on the fly),
//   B = the 2x2 real form [[wr, wi], [-wi, wr]] of w_ftr  (prepared once per launch),
// so Re/Im z_ft(n) = Z[n][2t], Z[n][2t+1], then g(n) += Σ_t conj(U_ft(n))·z_ft(n).
// tcgen05.mma kind::tf32 with a 3xTF32 split (hi·hi + hi·lo + lo·hi) keeps fp32-level
// accuracy (tools/umma_probe.cu: 3.9e-7 relative L2).
//
// A CTA owns half a tile (128 table positions = one M=128 block) and a range of frequencies.
// At start it stages the half-tile's table rows of every batch antenna in shared memory (bulk
// copies), so the phasor work reads shared memory only. K runs in chunks of 16 receivers:
// 512 threads (4 per voxel row) generate the A chunk into one of two shared-memory stages,
// B chunks arrive by bulk copy, and one thread issues the MMAs into one of two TMEM regions per
// frequency. The epilogue of frequency f-1 (tcgen05.ld, conj(U) phasors, complex MACs) runs
// while the tensor core works on frequency f. Each CTA publishes its half-tile partial through
// the flat adjoint's chunk combine (adj_epilogue), which applies the prox.

#ifndef NFGPU_TC
#define NFGPU_TC 1
#endif
constexpr int TC_CW = 16;                     // compute warps (4 per TMEM lane quarter)
constexpr int TC_CT = TC_CW * 32;             // compute threads
constexpr int TC_THREADS = TC_CT + 64;        // + B-loader warp + MMA warp
constexpr int TC_SUB = TC_CT / 128;           // compute threads per voxel row
constexpr int TC_RCH = 8;                     // receivers per pipeline step (K = 16 reals = two MMAs of K = 8)
constexpr int TC_NS = 4;                      // adjoint pipeline stages (at most; fewer when the table is large)
#ifndef NFGPU_TCF_NS
#define NFGPU_TCF_NS 2
#endif
#ifndef NFGPU_TCF_PROBE  // diagnostics only: 1 = skip the forward MMAs, 2 = skip the forward operand generation
#define NFGPU_TCF_PROBE 0
#endif
#ifndef NFGPU_TCF_VPS
#define NFGPU_TCF_VPS 16
#endif
constexpr int TCF_NS = NFGPU_TCF_NS;          // forward pipeline stages
constexpr int TCF_GW = 12;                    // forward generation warps (warps 12..15 drain TMEM)
constexpr int TC_NMAX = 128;                  // max padded 2·n_t (TMEM: 2 regions × N ≤ 256 columns)
constexpr uint32_t TC_A_BYTES = 128 * 2 * TC_RCH * 4;  // one of hi/lo: 8 KB
constexpr uint32_t TC_SMEM_MAX = 227 * 1024;
constexpr int TC_RX_MAX = 256;                     // receivers of a tensor-core batch (phase parameter slots)
constexpr int TC_ANT_MAX = TC_NMAX / 2 + TC_RX_MAX;  // batch antennas (tx <= TC_NMAX / 2 = 64)

// dynamic shared-memory layout of adj_tc_kernel (bytes), from the batch shape
struct TcLayout {
  uint32_t a_off, b_off, b_stage, tab_off, d0_off, par_off, bar_off, bytes;
  __host__ __device__ TcLayout(int npad, int nant, int ns = TC_NS) {
    a_off = 0;                                   // [stage][hi, lo][128 x 16]
    b_off = ns * 2 * TC_A_BYTES;                 // [stage][hi, lo][npad x 16]
    b_stage = (uint32_t)npad * 2 * TC_RCH * 4 * 2;
    tab_off = b_off + ns * b_stage;              // [antenna slot][δ 128 | 1/d 128]
    d0_off = tab_off + (uint32_t)nant * 1024;    // [TC_ANT_MAX] fp64 (batch antennas)
    par_off = d0_off + TC_ANT_MAX * 8;           // rx [2][kr 256 | br 256], tx [2][kt 64 | bt 64]
    bar_off = par_off + (1024 + 256) * 4;        // 3·NS + 4 mbarriers + TMEM base
    bytes = bar_off + (3 * TC_NS + 6) * 8;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle (canonical UMMA layout): 8-row x 16-B core matrices; byte offset of
// element (row, k) of a [rows][K] operand
__host__ __device__ __forceinline__ uint32_t kmaj(int row, int k, int rows) {
  return (uint32_t)((k >> 2) * (rows >> 3) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// round to the nearest tf32, ties away from zero (cvt.rna.tf32.f32 for finite x; ptxas expands that
// instruction with an inf/nan check, this is two integer ops)
__device__ __forceinline__ float tf32_round(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// amplitude-weighted one-sided phasor of one voxel: amp·(cos x, sgn·sin x), x = b + k·δ
template <bool EXACT>
__device__ __forceinline__ void phasor1(float k, float b, float dl, float amp, float sgn, float& re, float& im) {
  float x = fmaf(k, dl, b);
  if (EXACT) x = (x - ((x + 12582912.0f) - 12582912.0f)) * 6.28318530717958647692f;
  float s, c;
  __sincosf(x, &s, &c);
  re = amp * c;
  im = amp * sgn * s;
}

// two phasors at once on packed pairs: amp·(cos x, sin x), x = b + k·δ (sgn +1)
template <bool EXACT>
__device__ __forceinline__ void phasor2(float2 k, float2 b, float2 dl, float2 amp, float2& re, float2& im) {
  float2 x = fma2(k, dl, b);
  if (EXACT) x = mul2(sub2(x, sub2(add2(x, bc(12582912.0f)), bc(12582912.0f))), bc(6.28318530717958647692f));
  float2 sn, cs;
  __sincosf(x.x, &sn.x, &cs.x);
  __sincosf(x.y, &sn.y, &cs.y);
  re = mul2(amp, cs);
  im = mul2(amp, sn);
}

// B images of every (batch frequency, K chunk): [hi | lo] x [npad rows][32 k] in the smem layout
__global__ void tc_bprep_kernel(StructArgs sa, const float2* __restrict__ wrec, int npad, int nch,
                                float* __restrict__ out) {
  const int fi = blockIdx.x / nch, c = blockIdx.x - fi * nch;
  constexpr int KC = 2 * TC_RCH;
  float* img = out + (size_t)blockIdx.x * npad * KC * 2;
  for (int idx = threadIdx.x; idx < npad * KC; idx += blockDim.x) {
    const int n = idx / KC, k = idx - n * KC;
    const int t = n >> 1, cp = n & 1, q = k >> 1, cc = k & 1, r = c * TC_RCH + q;
    float v = 0.f;
    if (t < sa.nt && r < sa.nr) {
      const float2 w = wrec[((size_t)fi * sa.nt + t) * sa.nr + r];
      v = cc == 0 ? (cp == 0 ? w.x : w.y) : (cp == 0 ? -w.y : w.x);
    }
    const float h = tf32_round(v);
    const uint32_t o = kmaj(n, k, npad) >> 2;
    img[o] = h;
    img[npad * KC + o] = v - h;
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Warp-specialised: warps 0..7 generate A stages, warps 8..15 run the epilogue (two per TMEM
// lane quarter), warp 16 loads B, warp 17 issues the MMAs. Barriers: afull/sfree/bfull per
// stage, zfull/zfree per TMEM region; each role keeps its own per-frequency side parameters.
template <bool PROX, bool EXACT>
__global__ void __launch_bounds__(TC_THREADS, 1) adj_tc_kernel(AdjArgs<float> a, StructArgs sa,
                                                               const double* __restrict__ kd,
                                                               const float* __restrict__ bimg, int npad, int nch,
                                                               int fch, int ns) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const TcLayout ly(npad, sa.nt + sa.nr, ns);
  const Geo& g = a.g;
  const int tid = threadIdx.x, w = tid >> 5, L = tid & 31;
  // CTA = (tile, half hb, frequency chunk fc); it is chunk hb·fch + fc of the tile for adj_epilogue
  const int tile = blockIdx.x / (2 * fch), rem = blockIdx.x - tile * 2 * fch, hb = rem / fch, fc = rem - hb * fch;
  double* d0 = reinterpret_cast<double*>(sm + ly.d0_off);
  float* tsm = reinterpret_cast<float*>(sm + ly.tab_off);  // slot: δ[128], 1/d[128]; tx slots then rx slots
  float* par = reinterpret_cast<float*>(sm + ly.par_off);  // rx [2][kr 256 | br 256], tx [2][kt 64 | bt 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ly.bar_off);
  uint64_t *afull = bars, *sfree = bars + TC_NS, *bfull = bars + 2 * TC_NS, *zfull = bars + 3 * TC_NS,
           *zfree = bars + 3 * TC_NS + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3 * TC_NS + 4);
  const float* tabt = a.tab + (size_t)tile * g.A * TABW + hb * 128;
  const int nant = sa.nt + sa.nr;
  if (tid < TC_CT) {  // the half tile's table rows of every batch antenna (per-thread cp.async)
    for (int i = tid; i < nant * 64; i += TC_CT) {
      const int sl = i >> 6, part = i & 63, blk = part >> 5, q = part & 31;
      const int ant = sl < sa.nt ? sa.ts[sl] : g.T + sa.rs[sl - sa.nt];
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(tsm + sl * 256 + blk * 128 + q * 4)),
                   "l"(tabt + (size_t)ant * TABW + blk * TILE + q * 4)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int i = tid; i < nant; i += TC_CT)  // fp64 anchors per batch slot: no global index loads later
      d0[i] = a.D0[(size_t)tile * g.A + (i < sa.nt ? sa.ts[i] : g.T + sa.rs[i - sa.nt])];
  }
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&afull[i], TC_CW / 2);
      mbar_init(&sfree[i], 1);
      mbar_init(&bfull[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&zfull[i], 1);
      mbar_init(&zfree[i], TC_CW / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == TC_CW + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int f0 = (int)(((long long)sa.nf * fc) / fch), f1 = (int)(((long long)sa.nf * (fc + 1)) / fch);
  const int nfl = f1 - f0, nsteps = nfl * nch;
  const uint32_t bbytes = ly.b_stage;
  constexpr int HT = TC_CT / 2;  // threads per role

  if (w == TC_CW) {  // ---------------- B loader
    if (L == 0)
      for (int s = 0, st = 0, k = 0, fi = f0, c = 0; s < nsteps; ++s) {  // stage st, its use k; batch row fi, chunk c
        if (k > 0) mbar_wait(&sfree[st], (k - 1) & 1);
        mbar_expect(&bfull[st], bbytes);
        bulk_g2s(sm + ly.b_off + st * bbytes, bimg + ((size_t)fi * nch + c) * (bbytes / 4), bbytes, &bfull[st]);
        if (++st == ns) st = 0, ++k;
        if (++c == nch) c = 0, ++fi;
      }
  } else if (w == TC_CW + 1) {  // ---------------- MMA issuer
    if (L == 0) {
      const uint32_t idesc = umma_idesc_tf32(128, npad), lboB = (uint32_t)(npad >> 3) * 128;
      for (int s = 0, st = 0, k = 0, fl = 0, c = 0; s < nsteps; ++s) {
        mbar_wait(&afull[st], k & 1);
        mbar_wait(&bfull[st], k & 1);
        if (c == 0 && fl >= 2) mbar_wait(&zfree[fl & 1], ((fl - 2) >> 1) & 1);  // region read by epilogue(fl-2)
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((fl & 1) * npad);
        const uint32_t a0 = smem_u32(sm + ly.a_off + st * 2 * TC_A_BYTES);
        const uint32_t b0 = smem_u32(sm + ly.b_off + st * bbytes);
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const int ah = pass == 2 ? 1 : 0, bh = pass == 1 ? 1 : 0;  // hi·hi, hi·lo, lo·hi
#pragma unroll
          for (int ks = 0; ks < 2 * TC_RCH / 8; ++ks) {
            const uint64_t ad = umma_desc(a0 + ah * TC_A_BYTES + ks * 2 * 2048, 2048, 128);
            const uint64_t bd = umma_desc(b0 + bh * (bbytes / 2) + ks * 2 * lboB, lboB, 128);
            umma_tf32(d, ad, bd, idesc, (c > 0 || pass > 0 || ks > 0) ? 1u : 0u);
          }
        }
        umma_commit(&sfree[st]);
        if (c == nch - 1) umma_commit(&zfull[fl & 1]);
        if (++st == ns) st = 0, ++k;
        if (++c == nch) c = 0, ++fl;
      }
    }
  } else if (w < TC_CW / 2) {  // ---------------- A generation: conj(V) of 8 receivers per step
    const int row = tid & 127, sub = tid >> 7;  // 2 threads per voxel row
    int st = 0, k = 0;                          // pipeline stage and its use count
    double kfn = nfl > 0 ? kd[sa.fs[f0]] : 0.0;
    for (int fl = 0; fl < nfl; ++fl) {
      float* kr = par + (fl & 1) * 512;
      float* br = kr + 256;
      const double kf = kfn;
      if (fl + 1 < nfl) kfn = kd[sa.fs[f0 + fl + 1]];  // prefetch: lands while this frequency runs
      for (int q = tid; q < sa.nr; q += HT) side_params<float, EXACT>(kf, d0[sa.nt + q], kr[q], br[q]);
      named_bar(1, HT);
      for (int c = 0; c < nch; ++c) {
        if (k > 0) mbar_wait(&sfree[st], (k - 1) & 1);  // MMAs of step s - NS released the stage
        unsigned char* Ast = sm + ly.a_off + st * 2 * TC_A_BYTES;
#pragma unroll
        for (int qq = 0; qq < TC_RCH / 2; qq += 2) {  // two receivers (a packed pair) = one 16-B chunk of the row
          const int q = sub * (TC_RCH / 2) + qq;
          const int r0 = c * TC_RCH + q, r1 = r0 + 1;
          const int c0 = min(r0, sa.nr - 1), c1 = min(r1, sa.nr - 1);  // out-of-range partners get amplitude 0
          const float* p0 = tsm + (sa.nt + c0) * 256 + row;
          const float* p1 = tsm + (sa.nt + c1) * 256 + row;
          float2 re, im;
          phasor2<EXACT>(make_float2(kr[c0], kr[c1]), make_float2(br[c0], br[c1]), make_float2(p0[0], p1[0]),
                         make_float2(r0 < sa.nr ? p0[128] : 0.f, r1 < sa.nr ? p1[128] : 0.f), re, im);
          const float4 h = make_float4(tf32_round(re.x), tf32_round(im.x), tf32_round(re.y), tf32_round(im.y));
          const float2 l0 = sub2(make_float2(re.x, im.x), make_float2(h.x, h.y));
          const float2 l1 = sub2(make_float2(re.y, im.y), make_float2(h.z, h.w));
          const uint32_t off = kmaj(row, 2 * q, 128);
          *reinterpret_cast<float4*>(Ast + off) = h;
          *reinterpret_cast<float4*>(Ast + TC_A_BYTES + off) = make_float4(l0.x, l0.y, l1.x, l1.y);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (L == 0) mbar_arrive(&afull[st]);
        if (++st == ns) st = 0, ++k;
      }
    }
  } else {  // ---------------- epilogue: g += Σ_t conj(U_t)·z_t
    const int et = tid - HT, row = et & 127, sub = et >> 7;  // 2 threads per voxel row
    float2 g2r = make_float2(0.f, 0.f), g2i = g2r;          // even / odd transmitters, added at the end
    double kfn = nfl > 0 ? kd[sa.fs[f0]] : 0.0;
    for (int fl = 0; fl < nfl; ++fl) {
      float* kt = par + 1024 + (fl & 1) * 128;
      float* bt = kt + 64;
      const double kf = kfn;
      if (fl + 1 < nfl) kfn = kd[sa.fs[f0 + fl + 1]];
      for (int q = et; q < sa.nt; q += HT) side_params<float, EXACT>(kf, d0[q], kt[q], bt[q]);
      named_bar(2, HT);
      mbar_wait(&zfull[fl & 1], (fl >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + (uint32_t)((fl & 1) * npad) + ((uint32_t)(32 * (w & 3)) << 16);
      for (int t4 = sub; t4 * 4 < sa.nt; t4 += 2) {
        float z[8];
        tmem_ld8(base + t4 * 8, z);
#pragma unroll
        for (int j = 0; j < 4; j += 2) {  // transmitters t, t+1 as a packed pair
          const int t0 = t4 * 4 + j, t1 = t0 + 1;
          const int c0 = min(t0, sa.nt - 1), c1 = min(t1, sa.nt - 1);  // out-of-range partners get amplitude 0
          float2 ur, ui;
          phasor2<EXACT>(make_float2(kt[c0], kt[c1]), make_float2(bt[c0], bt[c1]),
                         make_float2(tsm[c0 * 256 + row], tsm[c1 * 256 + row]),
                         make_float2(t0 < sa.nt ? tsm[c0 * 256 + 128 + row] : 0.f,
                                     t1 < sa.nt ? tsm[c1 * 256 + 128 + row] : 0.f),
                         ur, ui);
          const float2 zr = make_float2(z[2 * j], z[2 * j + 2]), zi = make_float2(z[2 * j + 1], z[2 * j + 3]);
          g2r = fma2(ur, zr, fma2(make_float2(-ui.x, -ui.y), zi, g2r));
          g2i = fma2(ur, zi, fma2(ui, zr, g2i));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (L == 0) mbar_arrive(&zfree[fl & 1]);
    }
    const float gr = g2r.x + g2r.y, gi = g2i.x + g2i.y;
    // combine the two sub-threads; every MMA is complete, so the A stages are free
    float* cb = reinterpret_cast<float*>(sm + ly.a_off);  // [2][128][2]
    cb[(sub * 128 + row) * 2] = gr;
    cb[(sub * 128 + row) * 2 + 1] = gi;
    named_bar(2, HT);
    if (w == TC_CW / 2) {
      float Gr[V], Gi[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        Gr[v] = Gi[v] = 0.f;
        if ((v >> 2) == hb) {
          const int p = 4 * L + (v & 3);
          Gr[v] = cb[p * 2] + cb[(128 + p) * 2];
          Gi[v] = cb[p * 2 + 1] + cb[(128 + p) * 2 + 1];
        }
      }
      adj_epilogue<float, PROX>(a, tile, hb * fch + fc, a.CH, L, make_v(Gr), make_v(Gi), a.s_in, a.s_out);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == TC_CW + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ------------------------------------------------------------------ structured forward on tcgen05
//
// Per (half tile, f) the structured forward is a real GEMM (c64 only):
//   D[2t+c'][r] = Σ_k A[2t+c'][k] · B[r][k],   k = 2v + c over the half tile's 128 voxels,
//   A = the 2x2 real form [[Ur, -Ui], [Ui, Ur]] of U_ft(v),  B[r][2v] + j·B[r][2v+1] = V_fr(v)·s_v,
// so D[2t][r] + j·D[2t+1][r] = Σ_v U_ft(v)·V_fr(v)·s_v. Both operands are generated on the fly
// (3xTF32 split), 8 voxels (K = 16) per pipeline step. Warps 0..7 generate, warps 8..15 drain TMEM
// (the pair of lanes 2t, 2t+1 combined by a shuffle) into one partial per (half tile, channel),
// warp 17 issues the MMAs; fwd_reduce1/2 finish the sum over the 2·tiles partial rows.

constexpr int TCF_VPS = NFGPU_TCF_VPS;               // voxels per forward pipeline step
constexpr int TCF_KPS = 2 * TCF_VPS;                 // reals of K per step (4 MMAs of K = 8)
constexpr uint32_t TCF_A_BYTES = 128 * TCF_KPS * 4;  // one of hi/lo of an A stage
struct TcfLayout {
  uint32_t a_off, b_off, b_stage, s_off, tab_off, tab_buf, ant_off, d0_off, par_off, bar_off, bytes;
  // stream = false: the half tile's whole table is staged once; true: one step's slice at a time
  __host__ __device__ TcfLayout(int npr, int nant, bool stream) {
    a_off = 0;                                  // [stage][hi, lo][128 x KPS]
    b_off = TCF_NS * 2 * TCF_A_BYTES;           // [stage][hi, lo][npr x KPS]
    b_stage = (uint32_t)npr * TCF_KPS * 4 * 2;
    s_off = b_off + TCF_NS * b_stage;           // s of the half tile: [128] complex
    tab_off = s_off + 128 * 8;                  // table [voxel pair][slot, stride nant|1] (δ δ, 1/d 1/d):
    tab_buf = (uint32_t)(TCF_VPS / 2) * (nant | 1) * 16;  // whole half tile, or 2 x one step's slice
    ant_off = tab_off + (stream ? 2 * tab_buf : (uint32_t)(nant | 1) * 1024);  // [slot] antenna index
    d0_off = (ant_off + (uint32_t)nant * 4 + 7) & ~7u;
    par_off = d0_off + TC_ANT_MAX * 8;          // [2][k of slot 320 | b of slot 320]
    bar_off = par_off + 2 * 640 * 4;
    bytes = bar_off + (2 * TCF_NS + 6) * 8;
  }
};

template <bool EXACT, bool STREAM>
__global__ void __launch_bounds__(TC_THREADS, 1) fwd_tc_kernel(FwdArgs<float> a, StructArgs sa,
                                                               const double* __restrict__ kd, int npr, int fa, int fb,
                                                               int fch, float2* __restrict__ part) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const TcfLayout ly(npr, sa.nt + sa.nr, STREAM);
  const Geo& g = a.g;
  const int tid = threadIdx.x, w = tid >> 5, L = tid & 31;
  const int tile = blockIdx.x / (2 * fch), rem = blockIdx.x - tile * 2 * fch, hb = rem / fch, fc = rem - hb * fch;
  float2* ssm = reinterpret_cast<float2*>(sm + ly.s_off);
  double* d0 = reinterpret_cast<double*>(sm + ly.d0_off);
  // table [vp * TS + slot] = (δ of voxels 2vp, 2vp+1 | 1/d of 2vp, 2vp+1): the half tile's whole
  // table, staged once, or (STREAM) one pipeline step's slice, double-buffered, from L2 one step ahead
  float4* tvb = reinterpret_cast<float4*>(sm + ly.tab_off);
  int* antrow = reinterpret_cast<int*>(sm + ly.ant_off);
  float* par = reinterpret_cast<float*>(sm + ly.par_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ly.bar_off);
  uint64_t *afull = bars, *sfree = bars + TCF_NS, *zfull = bars + 2 * TCF_NS, *zfree = bars + 2 * TCF_NS + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * TCF_NS + 4);
  const float* tabt = a.tab + (size_t)tile * g.A * TABW + hb * 128;
  const int nant = sa.nt + sa.nr, mrows = 2 * sa.nt;
  const int TS = nant | 1;  // odd slot stride: neighbouring voxels of one slot land in different banks
  uint32_t tcols = 32;
  while (tcols < 2u * npr) tcols <<= 1;
  if (tid < TC_CT) {
    for (int i = tid; i < nant; i += TC_CT) {  // antenna of each batch slot; fp64 anchors per slot
      const int ant = i < sa.nt ? sa.ts[i] : g.T + sa.rs[i - sa.nt];
      antrow[i] = ant;
      d0[i] = a.D0[(size_t)tile * g.A + ant];
    }
    if (!STREAM)  // the whole table: (slot, voxel pair) as two 8-byte async copies (δ pair, 1/d pair)
      for (int i = tid; i < nant * 64; i += TC_CT) {
        const int sl = i >> 6, vp = i & 63;
        const int ant = sl < sa.nt ? sa.ts[sl] : g.T + sa.rs[sl - sa.nt];
        const float* src = tabt + (size_t)ant * TABW + 2 * vp;
        const uint32_t d = smem_u32(tvb + vp * TS + sl);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 8), "l"(src + TILE) : "memory");
      }
    if (tid < 128) {  // s at the half tile's table positions
      int tx, ty, tz;
      tile_coords(g, tile, tx, ty, tz);
      const int p = hb * 128 + tid, Lp = (p & 127) >> 2, v = 4 * (p >> 7) + (p & 3);
      int x0, y, z;
      lane_voxel(tx, ty, tz, Lp, x0, y, z);
      const int x = x0 + v;
      float2 sv = make_float2(0.f, 0.f);
      if (x < g.nx && y < g.ny && z < g.nzs) {
        const size_t n = ((size_t)z * g.ny + y) * g.nx + x;
        sv = make_float2(a.s[2 * n], a.s[2 * n + 1]);
      }
      ssm[tid] = sv;
    }
    // zero the padding rows of every stage once (A rows >= 2 n_t, B rows >= n_r); generation never writes them
    for (int st = 0; st < TCF_NS; ++st)
      for (int hl = 0; hl < 2; ++hl) {
        float* A0 = reinterpret_cast<float*>(sm + ly.a_off + (st * 2 + hl) * TCF_A_BYTES);
        for (int i = tid; i < (128 - mrows) * TCF_KPS; i += TC_CT)
          A0[kmaj(mrows + i / TCF_KPS, i % TCF_KPS, 128) >> 2] = 0.f;
        float* B0 = reinterpret_cast<float*>(sm + ly.b_off + st * ly.b_stage + hl * (ly.b_stage / 2));
        for (int i = tid; i < (npr - sa.nr) * TCF_KPS; i += TC_CT)
          B0[kmaj(sa.nr + i / TCF_KPS, i % TCF_KPS, npr) >> 2] = 0.f;
      }
  }
  if (tid == 0) {
    for (int i = 0; i < TCF_NS; ++i) {
      mbar_init(&afull[i], TCF_GW);
      mbar_init(&sfree[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&zfull[i], 1);
      mbar_init(&zfree[i], TC_CW - TCF_GW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == TC_CW + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zero padding is read by the MMAs
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nwin = fb - fa;
  const int f0 = fa + (int)(((long long)nwin * fc) / fch), f1 = fa + (int)(((long long)nwin * (fc + 1)) / fch);
  const int nfl = f1 - f0;
  constexpr int SPF = 128 / TCF_VPS;  // pipeline steps per frequency
  const int nsteps = nfl * SPF;

  if (w == TC_CW + 1) {  // ---------------- MMA issuer
    if (L == 0) {
      const uint32_t idesc = umma_idesc_tf32(128, npr), lboB = (uint32_t)(npr >> 3) * 128;
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % TCF_NS, k = s / TCF_NS, fl = s / SPF, c = s % SPF;
        mbar_wait(&afull[st], k & 1);
        if (c == 0 && fl >= 2) mbar_wait(&zfree[fl & 1], ((fl - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((fl & 1) * npr);
        const uint32_t a0 = smem_u32(sm + ly.a_off + st * 2 * TCF_A_BYTES);
        const uint32_t b0 = smem_u32(sm + ly.b_off + st * ly.b_stage);
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const int ah = pass == 2 ? 1 : 0, bh = pass == 1 ? 1 : 0;
#pragma unroll
          for (int ks = 0; ks < TCF_KPS / 8; ++ks) {
            const uint64_t ad = umma_desc(a0 + ah * TCF_A_BYTES + ks * 2 * 2048, 2048, 128);
            const uint64_t bd = umma_desc(b0 + bh * (ly.b_stage / 2) + ks * 2 * lboB, lboB, 128);
#if NFGPU_TCF_PROBE != 1
            umma_tf32(d, ad, bd, idesc, (c > 0 || pass > 0 || ks > 0) ? 1u : 0u);
#endif
          }
        }
        umma_commit(&sfree[st]);
        if (c == SPF - 1) umma_commit(&zfull[fl & 1]);
      }
    }
  } else if (w >= TCF_GW && w < TC_CW) {  // ---------------- epilogue: drain TMEM of each frequency
    // rows 2t, 2t+1 (lane pair) -> one complex partial per (half tile, channel). The pair splits each
    // 16-receiver chunk 8/8, so every lane stores 8 complex (64 contiguous bytes).
    const int span = a.w1 - a.w0;
    float2* out = part + (size_t)(2 * tile + hb) * span - a.w0;
    const int q = w & 3, row = 32 * q + L, t = row >> 1, odd = row & 1;
    for (int fl = 0; fl < nfl; ++fl) {
      mbar_wait(&zfull[fl & 1], (fl >> 1) & 1);
      tc_fence_after();
      if (32 * q < mrows) {
        const uint32_t base = tmem + (uint32_t)((fl & 1) * npr) + ((uint32_t)(32 * q) << 16);
        const int jb = (f0 + fl) * sa.nt * sa.nr;
        for (int r16 = 0; r16 * 16 < sa.nr; ++r16) {
          uint32_t rr[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]),
                "=r"(rr[7]), "=r"(rr[8]), "=r"(rr[9]), "=r"(rr[10]), "=r"(rr[11]), "=r"(rr[12]), "=r"(rr[13]),
                "=r"(rr[14]), "=r"(rr[15])
              : "r"(base + r16 * 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float2 o[8];  // even lane: receivers 0..7 of the chunk, odd lane: 8..15
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float lo8 = __uint_as_float(rr[j]), hi8 = __uint_as_float(rr[j + 8]);
            const float mine = odd ? hi8 : lo8;
            const float other = __shfl_xor_sync(FULL, odd ? lo8 : hi8, 1);
            o[j] = odd ? make_float2(other, mine) : make_float2(mine, other);
          }
          const int r0 = r16 * 16 + 8 * odd;
          if (t < sa.nt) {
            float2* dst = out + jb + t * sa.nr + r0;
            if (r0 + 8 <= sa.nr && ((sa.nr & 1) == 0)) {
#pragma unroll
              for (int j = 0; j < 8; j += 2)
                *reinterpret_cast<float4*>(dst + j) = make_float4(o[j].x, o[j].y, o[j + 1].x, o[j + 1].y);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (r0 + j < sa.nr) dst[j] = o[j];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (L == 0) mbar_arrive(&zfree[fl & 1]);
    }
  } else if (w < TCF_GW) {  // ---------------- generation: U (A operand) and W = V·s (B operand)
    // One item = (antenna, voxel pair) of a step; the thread computes both voxels. The first gu
    // warps take the U items (transmitters), the others the W items (receivers), in proportion
    // to n_t : n_r; lanes run over consecutive antennas (conflict-free table reads). Items go two
    // at a time with clamped, branch-free loads and math so their latency chains interleave;
    // only the stores of a padding item are skipped. A U item writes rows 2t, 2t+1 of A
    // ([[Ur, -Ui], [Ui, Ur]] form), a W item row r of B; hi and lo of the 3xTF32 split.
    constexpr int VP = TCF_VPS / 2;
    const int gu = min(TCF_GW - 1, max(1, (TCF_GW * sa.nt + (sa.nt + sa.nr) / 2) / (sa.nt + sa.nr)));
    const bool isU = w < gu;
    const int gthreads = 32 * (isU ? gu : TCF_GW - gu), gtid = isU ? tid : tid - 32 * gu;
    const int nant_k = isU ? sa.nt : sa.nr, nk = nant_k * VP;  // items of this kind
    const int slot0 = isU ? 0 : sa.nt;
    // item i = vp · nant_k + a; a thread's items advance by gthreads: (a, vp) += (dr, dq) with carry
    const int dq = gthreads / nant_k, dr = gthreads - dq * nant_k;
    const int a_first = gtid % nant_k, vp_first = gtid / nant_k;
    // one step's table slice: (slot, voxel pair) as two 8-byte copies (δ pair, 1/d pair)
    auto stage_slice = [&](int c, int buf) {
      float4* dst = tvb + buf * (ly.tab_buf / 16);
      for (int i = tid; i < nant * VP; i += TCF_GW * 32) {
        const int sl = i / VP, vp = i - sl * VP;
        const float* src = tabt + (size_t)antrow[sl] * TABW + c * TCF_VPS + 2 * vp;
        const uint32_t d = smem_u32(dst + vp * TS + sl);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 8), "l"(src + TILE) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (STREAM && nfl > 0) stage_slice(0, 0);
    double kfn = nfl > 0 ? kd[sa.fs[f0]] : 0.0;
    for (int fl = 0; fl < nfl; ++fl) {
      float* kp = par + (fl & 1) * 640;  // [slot] k, then [slot] b at +320
      const double kf = kfn;
      if (fl + 1 < nfl) kfn = kd[sa.fs[f0 + fl + 1]];  // prefetch: lands while this frequency runs
      for (int q = tid; q < nant; q += TCF_GW * 32) side_params<float, EXACT>(kf, d0[q], kp[q], kp[320 + q]);
      if (!STREAM) named_bar(1, TCF_GW * 32);
      for (int c = 0; c < SPF; ++c) {
        const int s = fl * SPF + c, st = s % TCF_NS, k = s / TCF_NS;
        if (STREAM) {  // this step's slice has landed for every thread, and every thread is done with
                       // step s-1 (its slice buffer and the previous frequency's parameters are free)
          asm volatile("cp.async.wait_all;" ::: "memory");
          named_bar(1, TCF_GW * 32);
          if (s + 1 < nsteps) stage_slice((c + 1) % SPF, (s + 1) & 1);
        }
        const float4* tv = STREAM ? tvb + (s & 1) * (ly.tab_buf / 16) : tvb + c * VP * TS;
        if (k > 0) mbar_wait(&sfree[st], (k - 1) & 1);
        unsigned char* Ast = sm + ly.a_off + st * 2 * TCF_A_BYTES;
        unsigned char* Bst = sm + ly.b_off + st * ly.b_stage;
        int an = a_first, vn = vp_first;
        for (int i0 = gtid; i0 < (NFGPU_TCF_PROBE == 2 ? 0 : nk); i0 += 2 * gthreads) {
          int ai[2], vi[2];
          bool ok[2];
          float4 e[2];
          float kk[2], bb[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            ok[u] = i0 + u * gthreads < nk;
            ai[u] = ok[u] ? an : ai[0];  // a padding item recomputes item 0; its stores are skipped
            vi[u] = ok[u] ? vn : vi[0];
            an += dr;
            vn += dq;
            if (an >= nant_k) an -= nant_k, ++vn;
            e[u] = tv[vi[u] * TS + slot0 + ai[u]];
            kk[u] = kp[slot0 + ai[u]];
            bb[u] = kp[320 + slot0 + ai[u]];
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int a_ = ai[u], vp = vi[u];
            float2 re, im;  // amp·(cos x, sin x) of voxels 2vp, 2vp+1; the phasor is re − j·im
            phasor2<EXACT>(bc(kk[u]), bc(bb[u]), make_float2(e[u].x, e[u].y), make_float2(e[u].z, e[u].w), re, im);
            if (isU) {  // U = re − j·im: row 2t (Ur, −Ui, ..) = (re, im, ..), row 2t+1 (Ui, Ur, ..)
              const float4 r0 = make_float4(re.x, im.x, re.y, im.y);
              const float4 h0 = make_float4(tf32_round(r0.x), tf32_round(r0.y), tf32_round(r0.z), tf32_round(r0.w));
              const float4 l0 = make_float4(r0.x - h0.x, r0.y - h0.y, r0.z - h0.z, r0.w - h0.w);
              if (ok[u]) {
                unsigned char* p0 = Ast + kmaj(2 * a_, 4 * vp, 128);
                *reinterpret_cast<float4*>(p0) = h0;
                *reinterpret_cast<float4*>(p0 + 16) = make_float4(-h0.y, h0.x, -h0.w, h0.z);
                *reinterpret_cast<float4*>(p0 + TCF_A_BYTES) = l0;
                *reinterpret_cast<float4*>(p0 + TCF_A_BYTES + 16) = make_float4(-l0.y, l0.x, -l0.w, l0.z);
              }
            } else {  // W = (re − j·im)·s
              const float4 sv = *reinterpret_cast<const float4*>(ssm + c * TCF_VPS + 2 * vp);
              const float4 q = make_float4(re.x * sv.x + im.x * sv.y, re.x * sv.y - im.x * sv.x,
                                           re.y * sv.z + im.y * sv.w, re.y * sv.w - im.y * sv.z);
              const float4 h = make_float4(tf32_round(q.x), tf32_round(q.y), tf32_round(q.z), tf32_round(q.w));
              if (ok[u]) {
                unsigned char* p0 = Bst + kmaj(a_, 4 * vp, npr);
                *reinterpret_cast<float4*>(p0) = h;
                *reinterpret_cast<float4*>(p0 + ly.b_stage / 2) = make_float4(q.x - h.x, q.y - h.y, q.z - h.z, q.w - h.w);
              }
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (L == 0) mbar_arrive(&afull[st]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == TC_CW + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// sorted-order bookkeeping of a structured batch: position j = (fi·nt + ti)·nr + ri is
// both the work order and the subset order (ascending channel id)
__global__ void struct_prep_kernel(StructArgs sa, int T, int R, int* __restrict__ sm, int* __restrict__ spos,
                                   int* __restrict__ sf) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int tr = sa.nt * sa.nr;
  if (j >= sa.nf * tr) return;
  const int fi = j / tr, rem = j - fi * tr, ti = rem / sa.nr, ri = rem - ti * sa.nr;
  const int f = sa.fs[fi];
  sm[j] = sa.rs[ri] + R * (sa.ts[ti] + T * f);
  spos[j] = j;
  sf[j] = f;
}

// level 1: tmp[seg][j] = Σ_{x in seg} part[x][j] (fp64, fixed order)
template <typename Real>
__global__ void fwd_reduce1_kernel(const Real* __restrict__ part, int nx, int span, int nseg,
                                   double2* __restrict__ tmp) {
  pdl_wait_and_release();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  if (j >= span) return;
  const int x0 = (int)(((long long)nx * seg) / nseg), x1 = (int)(((long long)nx * (seg + 1)) / nseg);
  double sr = 0, si = 0;
  for (int x = x0; x < x1; ++x) {
    const R2<Real> v = reinterpret_cast<const R2<Real>*>(part)[(size_t)x * span + j];
    sr += (double)v.x;
    si += (double)v.y;
  }
  tmp[(size_t)seg * span + j] = make_double2(sr, si);
}
// level 2: y[spos[j]] = p_f/(4π) Σ_seg tmp[seg][j]
template <typename Real>
__global__ void fwd_reduce2_kernel(const double2* __restrict__ tmp, int span, int nseg, int w0,
                                   const int* __restrict__ sf, const int* __restrict__ spos,
                                   const double* __restrict__ pulse, Real* __restrict__ y) {
  pdl_wait_and_release();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= span) return;
  double sr = 0, si = 0;
  for (int s = 0; s < nseg; ++s) {
    const double2 v = tmp[(size_t)s * span + j];
    sr += v.x;
    si += v.y;
  }
  const int f = sf[w0 + j];
  const double pr = pulse[2 * f] / (4.0 * PI), pim = pulse[2 * f + 1] / (4.0 * PI);
  const int k = spos[w0 + j];
  y[2 * (size_t)k] = (Real)(pr * sr - pim * si);
  y[2 * (size_t)k + 1] = (Real)(pr * si + pim * sr);
}

// ------------------------------------------------------------------ peer all-reduce of the forward partials
//
// Multi-GPU voxel-slab sharding: A_B s = Σ_p A_B[:, slab_p] s[slab_p].
// Instead of the NCCL all-reduce of the 2·B forward reals that follows nf_forward, the last forward
// reduce kernel pushes its (pre-pulse, fp64) channel sums straight into every rank's receive buffer
// over NVLink/NVSwitch (CUDA IPC peer mappings), raises one flag per (source rank, block) on every
// rank, waits for the flags of all source ranks for its own block, and sums the world slots in rank
// order, so every rank gets the same bits and the result does not depend on arrival order.
// Per-block epoch counters (advanced once per launch, in lockstep on all ranks) make the flags
// monotone; the receive buffer is double-buffered on epoch parity, so a fast rank can run one
// iteration ahead without overwriting slots a slow rank is still reading.
// With gridDim.y > 1 the same kernel emulates gridDim.y ranks in one cooperative launch on one GPU
// (tests: every block of every emulated rank is co-resident, no launch waits on another launch).
constexpr int PEER_MAX = 8;
constexpr long long PEER_SPIN_LIMIT = 1LL << 26;  // ~seconds of polling, then report instead of hanging
struct PeerArgs {
  int world, rank0;                    // rank of blockIdx.y == 0 (production: this rank, gridDim.y = 1)
  int cap, nblk_cap;                   // receive slots per (parity, source) and flag slots per source
  int blk_base;                        // flag/epoch slot of blockIdx.x == 0 in this launch
  double2* recv[PEER_MAX];             // every rank's receive buffer as mapped here: [2][world][cap]
  unsigned long long* flag[PEER_MAX];  // every rank's flags as mapped here: [world][nblk_cap]
  const double2* tmp[PEER_MAX];        // per grid rank: level-1 segment sums [nseg][span]
  void* y[PEER_MAX];                   // per grid rank: output, subset order
  unsigned long long* epoch[PEER_MAX]; // per grid rank: per-block launch counters [nblk_cap]
  int* err;                            // per grid rank 0: set to 1 if a wait timed out
};
__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
// FROM_Y = false: fused with level 2 of the forward reduce (flat batches; windows start at multiples of
// 256 channels, so flag slot w0/256 + block is the same channel group on every rank whatever its window
// split). FROM_Y = true: a one-shot all-reduce of a finished y (structured batches, whose window
// boundaries depend on the slab): slots per 256 channels of y, no pulse, no scatter.
template <typename Real, bool FROM_Y>
__global__ void __launch_bounds__(256) fwd_reduce2_peer_kernel(PeerArgs pa, int span, int nseg, int w0,
                                                               const int* __restrict__ sf,
                                                               const int* __restrict__ spos,
                                                               const double* __restrict__ pulse) {
  pdl_wait_and_release();
  const int gr = blockIdx.y, rank = pa.rank0 + gr, W = pa.world;
  const int b = pa.blk_base + blockIdx.x;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = j < span;
  const unsigned long long e = pa.epoch[gr][b] + 1;
  const int par = (int)(e & 1ULL);
  double sr = 0, si = 0;
  if (act && FROM_Y) {
    const Real* y = reinterpret_cast<const Real*>(pa.y[gr]);
    sr = (double)y[2 * (size_t)(w0 + j)];
    si = (double)y[2 * (size_t)(w0 + j) + 1];
  } else if (act) {
    for (int s = 0; s < nseg; ++s) {
      const double2 v = pa.tmp[gr][(size_t)s * span + j];
      sr += v.x;
      si += v.y;
    }
  }
  if (act)
    for (int q = 0; q < W; ++q) pa.recv[q][((size_t)par * W + rank) * pa.cap + w0 + j] = make_double2(sr, si);
  __syncthreads();  // the block's pushes happen before any of its flags
  if (threadIdx.x < W) {
    __threadfence_system();
    st_release_sys(pa.flag[threadIdx.x] + (size_t)rank * pa.nblk_cap + b, e);
  }
  if (threadIdx.x < W) {  // thread q waits for source rank q's push of this block
    const unsigned long long* f = pa.flag[rank] + (size_t)threadIdx.x * pa.nblk_cap + b;
    long long spins = 0;
    while (ld_acquire_sys(f) < e) {
      if (++spins > PEER_SPIN_LIMIT) {
        atomicExch(pa.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  double tr = 0, ti = 0;
  if (act) {
    const double2* src = pa.recv[rank] + (size_t)par * W * pa.cap + w0 + j;
    for (int q = 0; q < W; ++q) {  // fixed rank order: identical bits on every rank
      const double2 v = __ldcg(src + (size_t)q * pa.cap);
      tr += v.x;
      ti += v.y;
    }
    if (FROM_Y) {
      Real* y = reinterpret_cast<Real*>(pa.y[gr]);
      y[2 * (size_t)(w0 + j)] = (Real)tr;
      y[2 * (size_t)(w0 + j) + 1] = (Real)ti;
    }
  }
  if (act && !FROM_Y) {
    const int f = sf[w0 + j];
    const double pr = pulse[2 * f] / (4.0 * PI), pim = pulse[2 * f + 1] / (4.0 * PI);
    const int k = spos[w0 + j];
    Real* y = reinterpret_cast<Real*>(pa.y[gr]);
    y[2 * (size_t)k] = (Real)(pr * tr - pim * ti);
    y[2 * (size_t)k + 1] = (Real)(pr * ti + pim * tr);
  }
  if (threadIdx.x == 0) pa.epoch[gr][b] = e;
}

// ------------------------------------------------------------------ elementwise utilities
template <typename Real>
__global__ void soft_threshold_kernel(const Real* __restrict__ v, Real* __restrict__ out, int64_t n,
                                      double alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double vr = v[2 * i], vi = v[2 * i + 1];
  const double mag = hypot(vr, vi);  // np.abs: no overflow / underflow of the squares (solver.py:237)
  const double sc = mag > alpha ? (mag - alpha) / mag : 0.0;
  out[2 * i] = (Real)(vr * sc);
  out[2 * i + 1] = (Real)(vi * sc);
}

// {Σ|a|², Σ(|b|-|a|)²} with one block and a fixed summation order
template <typename Real>
__global__ void __launch_bounds__(1024) magchange_kernel(const Real* __restrict__ a, const Real* __restrict__ b,
                                                          int64_t n, double* __restrict__ out) {
  __shared__ double sh[2][1024];
  double s0 = 0, s1 = 0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) {
    const double ma = hypot((double)a[2 * i], (double)a[2 * i + 1]);
    const double mb = hypot((double)b[2 * i], (double)b[2 * i + 1]);
    s0 += ma * ma;
    s1 += (mb - ma) * (mb - ma);
  }
  sh[0][threadIdx.x] = s0;
  sh[1][threadIdx.x] = s1;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sh[0][0];
    out[1] = sh[1][0];
  }
}

// ------------------------------------------------------------------ CTA-tile ("ct") flat kernels
//
// For plans whose whole per-tile table (all T + R antennas: A·2·TILE Reals, 64 KB for BASELINE Medium in c64)
// fits twice in shared memory, a CTA of CT_WARPS warps works on ONE tile at a time with every row of it
// resident, and its warps split the tile's channels. Every CTA owns a contiguous range of the tile-major
// (tile, sorted channel) pairs of the launch (one CTA per SM; the cuts equalise pairs + cost x pieces, ct_args),
// cut into pieces (tile, channel range). A piece's table rows and D0 row arrive with two bulk copies (TMA) on an
// mbarrier, double-buffered: the last warp done with piece i refills its buffer with piece i + 2. No warp
// stages tx groups or receiver rows, and no warp waits for a straggler of another tile.
//   forward: each (tile, channel) value is computed by one warp with the flat kernel's arithmetic and
//            transpose-reduce, so part[tile][j] is bit-identical to fwd_kernel's and subsets stay bit-exact.
//   adjoint: the last warp done with a piece sums the warps' partial gradients in warp order (shared memory) and
//            parks the piece's sum in global memory; after the last piece the CTA's warps run the pieces'
//            epilogues side by side (a tile cut across CTAs sums its pieces in piece order, adj_epilogue), so no
//            warp carries several epilogues' latency into the end of the phase.
constexpr int CT_WARPS = 16;
constexpr int CT_TBR = 16;    // forward transpose depth of the CTA-tile kernel (lane sums in the order of TBR = 8)
#ifndef NFGPU_CT_UNROLL
#define NFGPU_CT_UNROLL 4
#endif
constexpr int CT_UNROLL = NFGPU_CT_UNROLL;  // adjoint channel loop (runs are long here)
constexpr int CT_TGA = 16;  // adjoint: transmitters per run group (their index rides in 4 low mantissa bits of the record)

template <typename Real>
struct CtLayout {  // [mbarriers, counters | buffer 0 | buffer 1 | warp records ×CT_WARPS | union region]
  size_t tab_bytes, buf_bytes, off_buf, off_warp, warp_bytes, off_u, u_bytes, bytes;
  __host__ __device__ explicit CtLayout(int A) {
    tab_bytes = (size_t)A * TABW * sizeof(Real);
    buf_bytes = tab_bytes + (size_t)d0_slots(A) * sizeof(double) + 2 * TILE * sizeof(Real);  // table | D0 | s
    off_buf = 64;
    off_warp = off_buf + 2 * buf_bytes;
    warp_bytes = 34 * sizeof(R4<Real>) + 34 * sizeof(int2);
    off_u = off_warp + (size_t)CT_WARPS * warp_bytes;
    const size_t tb = (size_t)CT_WARPS * CT_TBR * 33 * sizeof(R2<Real>);  // forward: per-warp transpose buffers
    const size_t gs = (size_t)2 * CT_WARPS * 2 * TILE * sizeof(Real);   // adjoint: warp partials [2][warps]
    u_bytes = tb > gs ? tb : gs;
    bytes = off_u + u_bytes;
  }
};

constexpr int CT_GMAX = 160;  // CTAs a CtArgs can describe (148 SMs on a B200)
struct CtArgs {
  long long W;  // ntiles * span: tile-major (tile, sorted channel) pairs of the launch window (< 2^31)
  int span;     // channels of the window
  int G;        // CTAs (one per SM; the persistent loop's grid)
  int ns;       // forward: pieces whose iterate values fit the staging area behind the layout (ct_stage_bytes)
  // CTA b owns pairs [bnd[b], bnd[b + 1]) (bnd[0] = 0, bnd[G] = W; empty ranges only at the end). Equal ranges leave
  // the CTAs whose range cuts one more tile behind the others (a piece has a fixed cost: table wait, record start-up,
  // partial combine), so ct_args places the cuts to minimise the largest pairs + cost * pieces instead. Forward values
  // do not depend on the cuts; the adjoint's chunk sums do, and nf_adjoint_prox and the persistent loop build the
  // same CtArgs.
  int bnd[CT_GMAX + 1];
};
// the CTA's range [r0, r1) of pairs: its first tile and piece count
struct CtRange {
  int r0, r1;
  int t0, np;
};
__device__ __forceinline__ CtRange ct_range(const CtArgs& c, int b) {
  CtRange r;
  r.r0 = c.bnd[b];
  r.r1 = c.bnd[b + 1];
  r.t0 = (int)((unsigned)r.r0 / (unsigned)c.span);
  r.np = r.r1 > r.r0 ? (int)((unsigned)(r.r1 - 1) / (unsigned)c.span) - r.t0 + 1 : 0;
  return r;
}
// the first and last of the CTAs whose ranges share `tile`, from CTA b, one of them
__device__ __forceinline__ void ct_sharers(const CtArgs& c, int tile, int b, int& first, int& last) {
  const long long u0 = (long long)tile * c.span, u1 = u0 + c.span;
  first = last = b;
  while (first > 0 && c.bnd[first] > u0) --first;
  while (last + 1 < c.G && c.bnd[last + 1] < u1) ++last;
}
// piece i of the range: tile and window-relative channels [ja, jb)
__device__ __forceinline__ void ct_piece(const CtArgs& c, const CtRange& r, int i, int& tile, int& ja, int& jb) {
  tile = r.t0 + i;
  const int base = tile * c.span;  // W < 2^31
  ja = max(r.r0 - base, 0);
  jb = min(r.r1 - base, c.span);
}
// warp w's slice of the piece's channels
__device__ __forceinline__ void ct_slice(int ja, int jb, int w, int& c0, int& c1) {
  c0 = ja + (int)(((unsigned)(jb - ja) * (unsigned)w) / CT_WARPS);  // spans stay far below 2^27
  c1 = ja + (int)(((unsigned)(jb - ja) * (unsigned)(w + 1)) / CT_WARPS);
}

// Fill buffer `buf` with tile's table rows (bulk copy, lane 0), its D0 row and (forward) its iterate values in the
// lane-quad layout of ldv (plain loads by the 32 lanes). mbarrier `full` (33 arrivals: the expect_tx of lane 0 and
// every lane after its stores) completes when all of it has landed.
template <typename Real>
__device__ __forceinline__ void ct_produce_table(const Geo& g, const Real* __restrict__ tab,
                                                 const double* __restrict__ D0, unsigned char* buf, uint64_t* full,
                                                 int tile, int L) {
  const CtLayout<Real> lay(g.A);
  double* d0 = reinterpret_cast<double*>(buf + lay.tab_bytes);
  // (an even antenna count keeps the tile's D0 row 16-byte aligned and sized: it rides a second bulk copy, and the
  // producing warp waits for no load)
  const bool d0_bulk = (g.A & 1) == 0;
  if (L == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the old piece before the copy
    const uint32_t d0_bytes = d0_bulk ? (uint32_t)g.A * (uint32_t)sizeof(double) : 0u;
    mbar_expect(full, (uint32_t)lay.tab_bytes + d0_bytes);
    bulk_g2s(buf, tab + (size_t)tile * g.A * TABW, (uint32_t)lay.tab_bytes, full);
    if (d0_bulk) bulk_g2s(d0, D0 + (size_t)tile * g.A, d0_bytes, full);
  }
  if (!d0_bulk)
    for (int i = L; i < g.A; i += 32) d0[i] = D0[(size_t)tile * g.A + i];
}
// the iterate values of `tile` in the lane-quad layout of ldv, into ss[2 * TILE]
template <typename Real, bool LOOP>
__device__ __forceinline__ void ct_stage_s(const Geo& g, const Real* __restrict__ sv, Real* ss, int tile, int L) {
  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(tx, ty, tz, L, x0, y, z);
  constexpr int QD = 16 / (int)sizeof(Real);
  const size_t n0 = ((size_t)z * g.ny + y) * g.nx + x0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const bool ok = x0 + v < g.nx && y < g.ny && z < g.nzs;
    Real re = 0, im = 0;
    if (ok) {
      re = LOOP ? __ldcg(sv + 2 * (n0 + v)) : sv[2 * (n0 + v)];
      im = LOOP ? __ldcg(sv + 2 * (n0 + v) + 1) : sv[2 * (n0 + v) + 1];
    }
    const int e = (v / QD) * 32 * QD + L * QD + v % QD;
    ss[e] = re;
    ss[TILE + e] = im;
  }
}
template <typename Real, bool LOOP>
__device__ __forceinline__ void ct_produce(const Geo& g, const Real* __restrict__ tab, const double* __restrict__ D0,
                                           const Real* __restrict__ sv, unsigned char* buf, uint64_t* full, int tile,
                                           int L, bool with_s) {
  ct_produce_table<Real>(g, tab, D0, buf, full, tile, L);
  if (with_s) {
    const CtLayout<Real> lay(g.A);
    ct_stage_s<Real, LOOP>(g, sv, reinterpret_cast<Real*>(buf + lay.tab_bytes + (size_t)d0_slots(g.A) * sizeof(double)),
                           tile, L);
  }
  mbar_arrive(full);
}

// Channel records of one batch of 32 (lane L <-> sorted position jb + L) as build_records, with the prefetch of
// the NEXT batch at an explicit position (pf, pf_end): the next batch of this slice, or the first batch of the
// warp's slice of the next piece.
template <typename Real, bool EXACT>
__device__ __forceinline__ unsigned ct_records(const Geo& g, const WarpSmem<Real>& ws, const ChanRec* __restrict__ crec,
                                               const R2<Real>* __restrict__ wrec, int nb, int pf, int pf_end, int L,
                                               int& carry, ChanRec& nxt, R2<Real>& nxtw) {
  const ChanRec cr = nxt;
  const R2<Real> w = nxtw;
  if (pf + L < pf_end) {
    nxt = crec[pf + L];
    if (wrec) nxtw = wrec[pf + L];
  }
  int key = -1, toff = 0;
  if (L < nb) {
    // Every tx row is resident, so runs need not follow the plan's tx groups. forward (no wrec): the record carries
    // the row's full offset and a run is a receiver (group 0 for all). adjoint: the record is full, and the tx index
    // within a group of CT_TGA = 16 rides in the 2 low mantissa bits of the phase offset and of the residual's real
    // part (a relative 2^-22 of that weight in c64): 4x fewer, longer runs than with the plan's groups of 4.
    const int t = pk_t(cr.pk), r = pk_r(cr.pk), tg = wrec ? t / CT_TGA : 0;
    const int tin = wrec ? t % CT_TGA : t;
    const double x = cr.kd * (ws.d0[t] + ws.d0[g.T + r]);
    R4<Real> q;
    if constexpr (std::is_same<Real, float>::value) {
      if (EXACT) {
        q.x = cr.kf;
        q.y = (float)(x - rint(x));
      } else {
        q.x = (float)(2.0 * PI * cr.kd);
        q.y = (float)(2.0 * PI * (x - rint(x)));
      }
    } else {
      q.x = cr.kd;
      q.y = (Real)(x - rint(x));
    }
    toff = tin * TABW;
    if (wrec) {
      q.z = with_low2(w.x, tin >> 2);
      q.w = w.y;
      q.y = with_low2(q.y, tin & 3);
    } else {
      q.z = int_bits<Real>(toff);
      q.w = 0;
    }
    ws.rec[L] = q;
    key = r | (tg << 15);
  }
  int prev = __shfl_up_sync(FULL, key, 1);
  if (L == 0) prev = carry;
  const unsigned starts = __ballot_sync(FULL, L < nb && key != prev);
  carry = __shfl_sync(FULL, key, nb - 1);
  if (L < nb) {
    const unsigned later = L < 31 ? (starts >> (L + 1)) << (L + 1) : 0u;
    const int end = later ? __ffs(later) - 1 : nb;
    ws.rect[L] = make_int2(toff, key | (end << 24));
  }
  __syncwarp();
  return starts;
}

// One warp's slice [c0, c1) (absolute sorted positions) of a forward piece: fwd_unit's channel loop on resident rows.
template <typename Real, bool EXACT>
__device__ __forceinline__ void ct_fwd_slice(const Geo& g, const Real* __restrict__ tab_s, const Real* __restrict__ s_s,
                                             const WarpSmem<Real>& ws, R2<Real>* tb, const ChanRec* __restrict__ crec,
                                             int c0, int c1, int pn0, int pn1, R2<Real>* __restrict__ outl, int L,
                                             ChanRec& nxt) {
  constexpr int QD = 16 / (int)sizeof(Real);
  R2<Real> nxtw;
  nxtw.x = 0;
  nxtw.y = 0;
  QV<Real> dR, iR, shr, shi, nshr;
  zero(dR);
  zero(iR);
  zero(shr);
  zero(shi);
  zero(nshr);
  const Real* tsl = tab_s + L * QD;
  int carry = -1, cur_rr = -1;
  for (int jb = c0; jb < c1; jb += 32) {
    const int nb = min(32, c1 - jb);
    const bool more = jb + 32 < c1;
    const unsigned starts = ct_records<Real, EXACT>(g, ws, crec, nullptr, nb, more ? jb + 32 : pn0, more ? c1 : pn1, L,
                                                    carry, nxt, nxtw);
    for (int h0 = 0; h0 < nb; h0 += CT_TBR) {
      const int h1 = min(nb, h0 + CT_TBR);
      int c = h0;
      while (c < h1) {
        const int key = ws.rect[c].y;
        const int e = min(key >> 24, h1);
        if ((starts >> c) & 1u) {  // a new (rx, tx-group) run begins at c: rows straight from the resident table
          const int rr = key & 0x7fff, tg = (key >> 15) & 0x1ff;
          tsl = tab_s + (size_t)tg * g.Tg * TABW + L * QD;
          if (rr != cur_rr) {  // a new receiver (rx-major batches: once per receiver, not per tx group)
            cur_rr = rr;
            const Real* rrow = tab_s + (size_t)(g.T + rr) * TABW + L * QD;
            dR = ldv(rrow);
            iR = ldv(rrow + TILE);
            // the iterate from shared memory at every receiver start (not held in registers)
            scale_s(iR, ldv(s_s + L * QD), ldv(s_s + TILE + L * QD), shr, shi, nshr);
          }
        }
        for (; c + 1 < e; c += 2) {
          const R4<Real> q0 = ws.rec[c], q1 = ws.rec[c + 1];
          const int o0 = bits_int(q0.z), o1 = bits_int(q1.z);
          const QV<Real> dT0 = ldv(tsl + o0), iT0 = ldv(tsl + o0 + TILE);
          const QV<Real> dT1 = ldv(tsl + o1), iT1 = ldv(tsl + o1 + TILE);
          QV<Real> cs0, sn0, cs1, sn1;
          phasorv<EXACT, NFGPU_FWD_CIS>(q0.x, q0.y, dT0, dR, cs0, sn0);
          phasorv<EXACT, NFGPU_FWD_CIS>(q1.x, q1.y, dT1, dR, cs1, sn1);
          const R2<Real> p0 = fwd_part(iT0, cs0, sn0, shr, shi, nshr);
          const R2<Real> p1 = fwd_part(iT1, cs1, sn1, shr, shi, nshr);
          tb[(c - h0) * 33 + L] = p0;
          tb[(c + 1 - h0) * 33 + L] = p1;
        }
        if (c < e) {
          const R4<Real> q = ws.rec[c];
          const int off = bits_int(q.z);
          const QV<Real> dT = ldv(tsl + off), iT = ldv(tsl + off + TILE);
          QV<Real> cs, sn;
          phasorv<EXACT, NFGPU_FWD_CIS>(q.x, q.y, dT, dR, cs, sn);
          tb[(c - h0) * 33 + L] = fwd_part(iT, cs, sn, shr, shi, nshr);
          ++c;
        }
      }
      __syncwarp();
      // 16 rows, two lanes per row. The flat kernels (TBR = 8) sum a channel's 32 lane values as four sequential
      // 8-sums S0..S3 combined (S0 + S2) + (S1 + S3); lane (row, h) forms S_h and S_{h+2} here, their sum, and one
      // shuffle adds the halves: the same operations in the same order, so the same bits.
      static_assert(TBR == 8 && CT_TBR == 16, "the CTA-tile transpose reproduces the TBR = 8 summation order");
      const int row = L % CT_TBR, h = L / CT_TBR;
      R2<Real> S, Sb;
      S.x = S.y = Sb.x = Sb.y = 0;
#pragma unroll 8
      for (int l = 0; l < 8; ++l) {
        const R2<Real> ta = tb[row * 33 + h * 8 + l], tc = tb[row * 33 + (h + 2) * 8 + l];
        if constexpr (std::is_same<Real, float>::value) {
          S = add2(S, ta);
          Sb = add2(Sb, tc);
        } else {
          S.x += ta.x;
          S.y += ta.y;
          Sb.x += tc.x;
          Sb.y += tc.y;
        }
      }
      if constexpr (std::is_same<Real, float>::value) {
        S = add2(S, Sb);
      } else {
        S.x += Sb.x;
        S.y += Sb.y;
      }
      S.x += __shfl_down_sync(FULL, S.x, 16);
      S.y += __shfl_down_sync(FULL, S.y, 16);
      if (L < h1 - h0) outl[jb + h0] = S;
      __syncwarp();
    }
  }
}

// the last of the CTA's warps to finish piece i on buffer b (counter in shared memory; it resets it)
__device__ __forceinline__ bool ct_last(int* cnt, int L) {
  __threadfence_block();
  __syncwarp();
  int last = 0;
  if (L == 0) {
    last = atomicAdd(cnt, 1) == CT_WARPS - 1;
    if (last) *cnt = 0;
  }
  last = __shfl_sync(FULL, last, 0);
  if (last) __threadfence_block();
  return last != 0;
}

// The CTA's forward pieces (per-launch kernel and persistent loop). ph: per-thread mbarrier parities.
template <typename Real, bool EXACT, bool LOOP>
__device__ __forceinline__ void ct_forward(const FwdArgs<Real>& a, const CtArgs& c, unsigned char* smem,
                                           const Real* __restrict__ sv, const ChanRec* __restrict__ crec,
                                           unsigned& ph, bool pdl) {
  const Geo& g = a.g;
  const CtLayout<Real> lay(g.A);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  int* cnt = reinterpret_cast<int*>(smem + 16);
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const CtRange rg = ct_range(c, blockIdx.x);
  const int np = rg.np;
  int tile, ja, jb;
  // When the staging area behind the layout holds every piece's iterate values (c.ns pieces), the warps load them
  // side by side now and a table refill is two bulk copies: the warp that issues it waits for no load.
  const bool sst = np <= c.ns;
  Real* ss_all = reinterpret_cast<Real*>(smem + lay.bytes);
  if (w == 0)
    for (int q = 0; q < 2 && q < np; ++q) {
      ct_piece(c, rg, q, tile, ja, jb);
      ct_produce<Real, LOOP>(g, a.tab, a.D0, sv, smem + lay.off_buf + q * lay.buf_bytes, full + q, tile, L, !sst);
    }
  if (sst) {
    for (int q = w; q < np; q += CT_WARPS) {
      ct_piece(c, rg, q, tile, ja, jb);
      ct_stage_s<Real, LOOP>(g, sv, ss_all + (size_t)q * 2 * TILE, tile, L);
    }
    __syncthreads();
  }
  if (pdl) pdl_wait();
  WarpSmem<Real> ws;
  unsigned char* wr = smem + lay.off_warp + (size_t)w * lay.warp_bytes;
  ws.rec = reinterpret_cast<R4<Real>*>(wr);
  ws.rect = reinterpret_cast<int2*>(wr + 34 * sizeof(R4<Real>));
  ws.tside = ws.rslot = nullptr;
  R2<Real>* tb = reinterpret_cast<R2<Real>*>(smem + lay.off_u) + (size_t)w * CT_TBR * 33;
  for (int i = L; i < 34; i += 32) ws.rect[i] = make_int2(0, -1);
  ChanRec nxt;
  R2<Real> nxtw;
  int c0 = 0, c1 = 0;
  if (np > 0) {
    ct_piece(c, rg, 0, tile, ja, jb);
    ct_slice(ja, jb, w, c0, c1);
    prefetch_first<Real>(crec, nullptr, a.w0 + c0, a.w0 + c1, L, nxt, nxtw);
  }
  for (int q = 0; q < np; ++q) {
    const int b = q & 1;
    ct_piece(c, rg, q, tile, ja, jb);
    ct_slice(ja, jb, w, c0, c1);
    int pn0 = 0, pn1 = 0;
    if (q + 1 < np) {
      int t2, ja2, jb2;
      ct_piece(c, rg, q + 1, t2, ja2, jb2);
      ct_slice(ja2, jb2, w, pn0, pn1);
    }
    unsigned char* buf = smem + lay.off_buf + b * lay.buf_bytes;
    mbar_wait(full + b, (ph >> b) & 1u);
    ph ^= 1u << b;
    ws.d0 = reinterpret_cast<double*>(buf + lay.tab_bytes);
    const Real* s_s = sst ? ss_all + (size_t)q * 2 * TILE
                          : reinterpret_cast<const Real*>(buf + lay.tab_bytes + (size_t)d0_slots(g.A) * sizeof(double));
    R2<Real>* outl = reinterpret_cast<R2<Real>*>(a.part) + (size_t)tile * c.span - a.w0 + L;
    if (c0 < c1)
      ct_fwd_slice<Real, EXACT>(g, reinterpret_cast<const Real*>(buf), s_s, ws, tb, crec, a.w0 + c0, a.w0 + c1,
                                a.w0 + pn0, a.w0 + pn1, outl, L, nxt);
    else if (pn0 + L < pn1)
      nxt = crec[a.w0 + pn0 + L];
    if (ct_last(cnt + b, L) && q + 2 < np) {
      ct_piece(c, rg, q + 2, tile, ja, jb);
      ct_produce<Real, LOOP>(g, a.tab, a.D0, sv, buf, full + b, tile, L, !sst);
    }
  }
}

// One warp's slice of an adjoint piece: adj_unit's channel loop on resident rows; returns the flushed partial g.
template <typename Real, bool EXACT>
__device__ __forceinline__ void ct_adj_slice(const Geo& g, const Real* __restrict__ tab_s, const WarpSmem<Real>& ws,
                                             const ChanRec* __restrict__ crec, const R2<Real>* __restrict__ wrec,
                                             int c0, int c1, int pn0, int pn1, int L, ChanRec& nxt, R2<Real>& nxtw,
                                             QV<Real>& gr, QV<Real>& gi) {
  constexpr int QD = 16 / (int)sizeof(Real);
  QV<Real> hr, hi, dR, iR;
  zero(gr);
  zero(gi);
  zero(hr);
  zero(hi);
  zero(dR);
  zero(iR);
  const Real* tsl = tab_s + L * QD;
  int carry = -1, cur_rr = -1;
  for (int jb = c0; jb < c1; jb += 32) {
    const int nb = min(32, c1 - jb);
    const bool more = jb + 32 < c1;
    const unsigned starts = ct_records<Real, EXACT>(g, ws, crec, wrec, nb, more ? jb + 32 : pn0, more ? c1 : pn1, L,
                                                    carry, nxt, nxtw);
    int c = 0;
    while (c < nb) {
      const int key = ws.rect[c].y;
      const int e = key >> 24;
      if ((starts >> c) & 1u) {
        const int rr = key & 0x7fff, tg = (key >> 15) & 0x1ff;
        tsl = tab_s + (size_t)tg * CT_TGA * TABW + L * QD;
        if (rr != cur_rr) {  // a new receiver: g += h/d_R, its rows (rx-major batches: once per receiver)
          cur_rr = rr;
          flush(iR, hr, hi, gr, gi);
          const Real* rrow = tab_s + (size_t)(g.T + rr) * TABW + L * QD;
          dR = ldv(rrow);
          iR = ldv(rrow + TILE);
        }
      }
      R4<Real> q = ws.rec[c];
      int off = (low2(q.y) | (low2(q.z) << 2)) * TABW;
#pragma unroll CT_UNROLL
      for (; c < e; ++c) {
        const R4<Real> qn = ws.rec[c + 1];
        const int offn = (low2(qn.y) | (low2(qn.z) << 2)) * TABW;
        const QV<Real> dT = ldv(tsl + off), iT = ldv(tsl + off + TILE);
        QV<Real> cs, sn;
        phasorv<EXACT>(q.x, q.y, dT, dR, cs, sn);
        adj_acc(iT, cs, sn, q.z, q.w, hr, hi);
        q = qn;
        off = offn;
      }
    }
    __syncwarp();
  }
  flush(iR, hr, hi, gr, gi);
}

// The CTA's adjoint (+prox) pieces: slices as ct_forward; the last warp done with piece q combines the warps'
// partials (warp order) into slot q of this CTA's part of `cpart` ([CTAs][pmax][32 lanes][2V] Reals); after the
// last piece every piece's epilogue (adj_epilogue, chunk = its index among the CTAs sharing the tile) runs on its
// own warp.
template <typename Real, bool PROX, bool EXACT, bool LOOP>
__device__ __forceinline__ void ct_adjoint(const AdjArgs<Real>& a, const CtArgs& c, unsigned char* smem,
                                           const Real* __restrict__ s_in, Real* __restrict__ s_out,
                                           const ChanRec* __restrict__ crec, Real* __restrict__ cpart, int pmax,
                                           unsigned& ph, bool pdl) {
  const Geo& g = a.g;
  const CtLayout<Real> lay(g.A);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  int* cnt = reinterpret_cast<int*>(smem + 16);
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const CtRange rg = ct_range(c, blockIdx.x);
  const int np = rg.np;
  int tile, ja, jb;
  if (w == 0)
    for (int q = 0; q < 2 && q < np; ++q) {
      ct_piece(c, rg, q, tile, ja, jb);
      ct_produce_table<Real>(g, a.tab, a.D0, smem + lay.off_buf + q * lay.buf_bytes, full + q, tile, L);
      mbar_arrive(full + q);
    }
  WarpSmem<Real> ws;
  unsigned char* wr = smem + lay.off_warp + (size_t)w * lay.warp_bytes;
  ws.rec = reinterpret_cast<R4<Real>*>(wr);
  ws.rect = reinterpret_cast<int2*>(wr + 34 * sizeof(R4<Real>));
  ws.tside = ws.rslot = nullptr;
  for (int i = L; i < 34; i += 32) ws.rect[i] = make_int2(0, -1);
  using U16 = typename std::conditional<std::is_same<Real, float>::value, float4, double2>::type;
  constexpr int NU = 2 * V * (int)sizeof(Real) / 16, PU = 16 / (int)sizeof(Real);
  U16* gs = reinterpret_cast<U16*>(smem + lay.off_u);  // [2][CT_WARPS][NU][32] 16-byte quads
  U16* cp = reinterpret_cast<U16*>(cpart) + (size_t)blockIdx.x * pmax * NU * 32;  // [pmax][NU][32]
  ChanRec nxt;
  R2<Real> nxtw;
  int c0 = 0, c1 = 0;
  if (np > 0) {
    ct_piece(c, rg, 0, tile, ja, jb);
    ct_slice(ja, jb, w, c0, c1);
    prefetch_first<Real>(crec, nullptr, c0, c1, L, nxt, nxtw);
  }
  if (pdl) pdl_wait();
  if (np > 0 && c0 + L < c1) nxtw = a.wrec[c0 + L];
  for (int q = 0; q < np; ++q) {
    const int b = q & 1;
    ct_piece(c, rg, q, tile, ja, jb);
    ct_slice(ja, jb, w, c0, c1);
    int pn0 = 0, pn1 = 0;
    if (q + 1 < np) {
      int t2, ja2, jb2;
      ct_piece(c, rg, q + 1, t2, ja2, jb2);
      ct_slice(ja2, jb2, w, pn0, pn1);
    }
    unsigned char* buf = smem + lay.off_buf + b * lay.buf_bytes;
    NF_CHECK(tile >= 0 && tile < g.ntiles && 0 <= c0 && c0 <= c1 && c1 <= c.span && pn1 <= c.span,
             "adj piece q %d tile %d c0 %d c1 %d pn %d %d span %d\n", q, tile, c0, c1, pn0, pn1, c.span);
    mbar_wait(full + b, (ph >> b) & 1u);
    ph ^= 1u << b;
    ws.d0 = reinterpret_cast<double*>(buf + lay.tab_bytes);
    QV<Real> gr, gi;
    if (c0 < c1) {
      ct_adj_slice<Real, EXACT>(g, reinterpret_cast<const Real*>(buf), ws, crec, a.wrec, c0, c1, pn0, pn1, L, nxt,
                                nxtw, gr, gi);
    } else {
      zero(gr);
      zero(gi);
      if (pn0 + L < pn1) {
        nxt = crec[pn0 + L];
        nxtw = a.wrec[pn0 + L];
      }
    }
    {  // publish the warp's partial (interleaved re/im quads)
      Real t[2 * V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        t[2 * v] = get(gr, v);
        t[2 * v + 1] = get(gi, v);
      }
      U16* mine = gs + ((size_t)(b * CT_WARPS + w) * NU) * 32 + L;
#pragma unroll
      for (int u = 0; u < NU; ++u) mine[u * 32] = *reinterpret_cast<const U16*>(t + u * PU);
    }
    if (ct_last(cnt + b, L)) {  // combine in warp order, park the piece's sum, refill the buffer
      Real G[2 * V];
#pragma unroll
      for (int e = 0; e < 2 * V; ++e) G[e] = 0;
      for (int ww = 0; ww < CT_WARPS; ++ww) {
        const U16* src = gs + ((size_t)(b * CT_WARPS + ww) * NU) * 32 + L;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const U16 v4 = src[u * 32];
          const Real* tv = reinterpret_cast<const Real*>(&v4);
#pragma unroll
          for (int k = 0; k < PU; ++k) G[u * PU + k] += tv[k];
        }
      }
      NF_CHECK(q < pmax, "q %d pmax %d np %d b %d\n", q, pmax, np, (int)blockIdx.x);
#pragma unroll
      for (int u = 0; u < NU; ++u) cp[((size_t)q * NU + u) * 32 + L] = *reinterpret_cast<const U16*>(G + u * PU);
      if (q + 2 < np) {
        int t2, ja2, jb2;
        ct_piece(c, rg, q + 2, t2, ja2, jb2);
        ct_produce_table<Real>(g, a.tab, a.D0, buf, full + b, t2, L);
        mbar_arrive(full + b);
      }
    }
  }
  __syncthreads();  // every piece's sum is parked (global stores by this CTA's warps)
  for (int q = w; q < np; q += CT_WARPS) {
    ct_piece(c, rg, q, tile, ja, jb);
    Real Gr[V], Gi[V];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const U16 v4 = __ldcg(cp + ((size_t)q * NU + u) * 32 + L);
      const Real* tv = reinterpret_cast<const Real*>(&v4);
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        const int e = u * PU + k;
        if (e & 1)
          Gi[e >> 1] = tv[k];
        else
          Gr[e >> 1] = tv[k];
      }
    }
    const QV<Real> sgr = make_v(Gr), sgi = make_v(Gi);
    int first, lastc;
    ct_sharers(c, tile, (int)blockIdx.x, first, lastc);
    NF_CHECK(tile >= 0 && tile < g.ntiles && first <= (int)blockIdx.x && (int)blockIdx.x <= lastc && lastc < c.G,
             "tile %d first %d last %d b %d\n", tile, first, lastc, (int)blockIdx.x);
    adj_epilogue<Real, PROX, LOOP>(a, tile, (int)blockIdx.x - first, lastc - first + 1, L, sgr, sgi, s_in, s_out);
  }
}

__device__ __forceinline__ void ct_init(unsigned char* smem) {
  if (threadIdx.x == 0) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    mbar_init(full, 33);
    mbar_init(full + 1, 33);
    reinterpret_cast<int*>(smem + 16)[0] = 0;
    reinterpret_cast<int*>(smem + 16)[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

template <typename Real, bool EXACT>
__global__ void __launch_bounds__(CT_WARPS * 32, 1) fwd_ct_kernel(FwdArgs<Real> a, CtArgs c) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ct_init(smem_raw);
  unsigned ph = 0;
  ct_forward<Real, EXACT, false>(a, c, smem_raw, a.s, a.crec, ph, true);
}

template <typename Real, bool PROX, bool EXACT>
__global__ void __launch_bounds__(CT_WARPS * 32, 1) adj_ct_kernel(AdjArgs<Real> a, CtArgs c, Real* cpart, int pmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ct_init(smem_raw);
  unsigned ph = 0;
  ct_adjoint<Real, PROX, EXACT, false>(a, c, smem_raw, a.s_in, a.s_out, a.crec, cpart, pmax, ph, true);
}

// ------------------------------------------------------------------ persistent SPGM loop
//
// spgm_loop_kernel runs K SPGM iterations (solver.py:281-310) of a flat batch in ONE cooperative launch, one CTA
// per SM: the device-side loop for latency-bound configurations (BASELINE Small: 12 launches of ~3 us each per
// iteration otherwise). Per iteration, three phases between three grid barriers:
//   P1  forward(k): CTA-tile pieces (ct_forward) or warp units (fwd_unit, the body of fwd_kernel) -> part[tile][j].
//       One CTA (the last, "sorter") first draws iteration k+1's batch (index table row, or the Feistel sampler), sorts
//       its (key, position) keys by rank in shared memory (same order as the counting sort of nf_batch_prepare) and
//       writes the sorted channel records of parity (k+1) & 1, with {p_f, y_meas[m_j]} per sorted position
//   P2  both levels of the forward reduce and the residual records in one phase, per channel, on the other CTAs
//       (fwd_reduce1_kernel's, fwd_reduce2_kernel's and resid_kernel's sums in their order); the sorter reduces the
//       statistics of iteration k-1 (stats_reduce_kernel's tree), records them and tests the tolerance: a stop takes
//       effect after this phase's barrier (the forward and reduce of the iteration after the last one are
//       discarded), and the last iteration's statistics follow the loop
//   P3  adjoint(k) + prox: CTA-tile pieces (ct_adjoint) or warp units (adj_unit) -> s_out, per-tile statistics
// Every value is computed by the same code in the same order as the per-launch path, so the iterates are
// bit-identical to nf_batch_prepare + nf_forward + nf_adjoint_prox (tested). The time budget is checked on the
// device clock by the CTA that records the statistics and takes effect after the next barrier.
constexpr int LOOP_SORT_MAX = 4096;  // batches sorted in shared memory
constexpr int LOOP_REC = 6;          // per iteration: the 4 statistics, device time (ns since launch), spare

struct LoopArgs {
  KeyMap km;
  int M, B, K, nseg, hb;
  const int* __restrict__ idx_table;  // [K][B] (subset order) or null: Feistel sampler
  uint64_t seed, iter0;
  const double* __restrict__ kd;
  const double* __restrict__ pulse;
  const void* ymeas;
  int* sm;              // spgm_loop_kernel: sorted records [2 parities][B]
  int* spos;
  int* sf;
  double2* yrec;        // [2 parities][B][2]: {p_f, y_meas[m_j]} of sorted position j
  int ymeas_f64;        // y_meas is complex128
  ChanRec* crec;
  double2* tmp;
  double* dpart;
  double* stat_part;
  double tol;
  long long budget_ns;  // < 0: no time budget
  double eta_over_b, alpha;  // tiny_loop_kernel's prox (spgm_loop_kernel takes them from its AdjArgs)
  double* rec;          // [K][LOOP_REC]
  int* state;           // {iterations, reason: 0 max_iters / 1 tolerance / 2 time budget, stop flag}
  unsigned* bar;        // grid barrier arrival counter (grid_sync)
  int stage_tiles;      // the reduce phase stages a CTA's partials in shared memory, this many tiles at a time (0: no)
  int kwords;           // 32-bit words of the key-space bitmap of the P0 rank sort (0: pairwise ranks)
  int* ctr;             // work-unit counters {forward, adjoint}: warps fetch units past the first TW dynamically
  void* s_a;            // iteration k reads s_a (k even) or s_b (k odd) and writes the other
  void* s_b;
  size_t warp_bytes;
  void* ctpart;              // CTA-tile adjoint: parked piece sums [CTAs][ctpmax][32][2V]
  int ctpmax;
  const int* prev_state;     // chained launches: the previous launch's state; it stopped early -> run nothing
  int fold;                  // the latest iterate ends in s_a (an odd count copies s_b back; chained launches)
  unsigned long long* prof;  // diagnostics (NFGPU_LOOP_PROFILE): CTA 0's device clock at each phase boundary
  int prof_cta;              // ... and (NFGPU_LOOP_PROFILE=2) every CTA's at the ends of its forward and adjoint
};
constexpr int LOOP_PROF = 12;
constexpr int LOOP_PROF_CTA = 160;  // NFGPU_LOOP_PROFILE=2: also every CTA's forward and adjoint end (spgm_loop)

// Chained persistent launches (nf_spgm_loop_chained): the host enqueues launch j + 1 before it has read launch j's
// state. A launch whose predecessor stopped early (tolerance or budget) runs no iteration and forwards its reason.
__device__ __forceinline__ bool loop_skip(const LoopArgs& la) {
  if (!la.prev_state) return false;
  const int prev = *(volatile const int*)(la.prev_state + 1);
  if (prev != 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    la.state[0] = 0;
    la.state[1] = prev;
  }
  return prev != 0;
}
// ... and every launch ends with the latest iterate in s_a: after an odd count (written to s_b) all CTAs copy it
// back (every write to s_b happened before the last grid barrier, and nothing reads s_a any more)
template <typename Real>
__device__ __forceinline__ void loop_fold(const LoopArgs& la, int done, long long nvox) {
  if (!la.fold || !(done & 1)) return;
  const Real* src = reinterpret_cast<const Real*>(la.s_b);
  Real* dst = reinterpret_cast<Real*>(la.s_a);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * nvox; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// grid barrier (all CTAs co-resident: cooperative launch) on one monotonic arrival counter, zeroed by the host before
// every launch: thread 0 arrives with a release reduction (cumulative over the CTA's writes ordered before it by
// __syncthreads) and polls the counter with acquire loads until the n-th barrier's G arrivals are in. Every CTA
// counts its own barriers (`nbar`), so a barrier costs the reduction's trip to L2 and one poll, with no generation
// word to read first and no last arrival to publish it.
__device__ __forceinline__ void red_release_add_u32(unsigned* a, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& nbar) {
  __syncthreads();
  ++nbar;
  if (threadIdx.x == 0) {
    red_release_add_u32(bar, 1u);
    const unsigned target = nbar * gridDim.x;
    while ((int)(ld_acquire_u32(bar) - target) < 0) {
    }
  }
  __syncthreads();
}
// next work unit of a warp: the first TW units are assigned statically (unit = global warp index), later ones
// are fetched in launch order from a counter, like the hardware's CTA scheduler (balances unequal units)
__device__ __forceinline__ int next_unit(int* ctr, int TW, int L) {
  int u = 0;
  if (L == 0) u = atomicAdd(ctr, 1);
  return __shfl_sync(FULL, u, 0) + TW;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ int loop_index(const LoopArgs& la, int k, int i) {
  if (la.idx_table) return la.idx_table[(size_t)k * la.B + i];
  const uint64_t key = sample_key(la.seed, la.iter0 + (uint64_t)k);
  uint32_t x = (uint32_t)i;
  do {
    x = feistel(x, la.hb, key);
  } while (x >= (uint32_t)la.M);
  return (int)x;
}

// P0 of an iteration (one CTA): draw its batch and rank the keys (distinct) in shared memory, then write the B
// channel records in key order (the counting sort's order) to the records of parity k & 1. Ranks come from a
// bitmap of the key space and a prefix count of its words when the bitmap fits, else pairwise.
__device__ __forceinline__ void loop_sort(const LoopArgs& la, int k, int* scan_sh, unsigned char* smem_raw) {
  const int B = la.B;
  int* keys = reinterpret_cast<int*>(smem_raw);
  int* order = keys + LOOP_SORT_MAX;
  unsigned* bm = reinterpret_cast<unsigned*>(order + LOOP_SORT_MAX);
  int* pre = reinterpret_cast<int*>(bm + la.kwords);
  const bool bitmap = la.kwords > 0;
  if (bitmap)
    for (int i = threadIdx.x; i < la.kwords; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const int key = key_of(la.km, loop_index(la, k, i));
    keys[i] = key;
    if (bitmap) atomicOr(bm + (key >> 5), 1u << (key & 31));
  }
  __syncthreads();
  if (bitmap) {  // pre[w] = set bits in words < w
    const int per = (la.kwords + blockDim.x - 1) / blockDim.x, w0 = threadIdx.x * per;
    const int w1 = min(la.kwords, w0 + per);
    int cnt = 0;
    for (int q = w0; q < w1; ++q) cnt += __popc(bm[q]);
    int total;
    int run = block_excl_scan(cnt, scan_sh, total);
    for (int q = w0; q < w1; ++q) {
      pre[q] = run;
      run += __popc(bm[q]);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const int ki = keys[i];
    int r = 0;
    if (bitmap) {
      r = pre[ki >> 5] + __popc(bm[ki >> 5] & ((1u << (ki & 31)) - 1u));
    } else {
      for (int q = 0; q < B; ++q) r += keys[q] < ki;
    }
    order[r] = i;
  }
  __syncthreads();
  const size_t base = (size_t)(k & 1) * B;
  for (int j = threadIdx.x; j < B; j += blockDim.x) {
    const int pos = order[j], key = keys[pos];
    const int4 c = chan_of_key(la.km, key);
    la.sm[base + j] = c.z + la.km.R * (c.y + la.km.T * c.x);
    la.spos[base + j] = pos;
    ChanRec q;
    q.kd = la.kd[c.x];
    q.kf = (float)q.kd;
    q.pk = c.y | (c.z << 16);
    la.crec[base + j] = q;
    la.sf[base + j] = c.x;
    // what the residual record of position j needs (the reduce phase then has no dependent loads)
    const int m = c.z + la.km.R * (c.y + la.km.T * c.x);
    double yr, yi;
    if (la.ymeas_f64) {
      yr = reinterpret_cast<const double*>(la.ymeas)[2 * (size_t)m];
      yi = reinterpret_cast<const double*>(la.ymeas)[2 * (size_t)m + 1];
    } else {
      yr = (double)reinterpret_cast<const float*>(la.ymeas)[2 * (size_t)m];
      yi = (double)reinterpret_cast<const float*>(la.ymeas)[2 * (size_t)m + 1];
    }
    la.yrec[2 * (base + j)] = make_double2(la.pulse[2 * c.x], la.pulse[2 * c.x + 1]);
    la.yrec[2 * (base + j) + 1] = make_double2(yr, yi);
  }
  __syncthreads();
}

// statistics of iteration k (stats_reduce_kernel's tree, threads 0-255 of every CTA, the same bits everywhere),
// its record (CTA 0) and the time-budget flag; returns the relative magnitude change
__device__ __forceinline__ double loop_stats(const LoopArgs& la, int k, int ntiles, double (*red)[256], double* grp8,
                                             unsigned long long t0, bool writer) {
  if (threadIdx.x < 256) {
    double acc[4] = {0, 0, 0, 0};
    for (int i = threadIdx.x; i < ntiles; i += 256) {
      acc[0] += la.stat_part[(size_t)i * 4 + 0];
      acc[1] += la.stat_part[(size_t)i * 4 + 1];
      acc[3] += la.stat_part[(size_t)i * 4 + 3];
    }
    // resid_kernel's per-256-channel sums (lanes by xor tree, then the 8 warps in order) of iteration k's |y - y_meas|^2
    const double* e2 = reinterpret_cast<const double*>(la.tmp) + (size_t)(k & 1) * la.B;
    const int nd = (la.B + 255) / 256;
    for (int grp = 0; grp < nd; ++grp) {
      const int j = grp * 256 + (int)threadIdx.x;
      double e = j < la.B ? __ldcg(e2 + j) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
      if ((threadIdx.x & 31) == 0) grp8[threadIdx.x >> 5] = e;
      named_sync(3, 256);
      if ((int)threadIdx.x == (grp & 255)) {
        double t = 0;
        for (int i = 0; i < 8; ++i) t += grp8[i];
        acc[2] += t;
      }
      named_sync(3, 256);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = acc[q];
    named_sync(3, 256);
    for (int sh = 128; sh > 0; sh >>= 1) {
      if (threadIdx.x < sh)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + sh];
      named_sync(3, 256);
    }
  }
  __syncthreads();
  const double st0 = red[0][0], st1 = red[1][0];
  if (writer && threadIdx.x == 0) {
    double* r = la.rec + (size_t)k * LOOP_REC;
    r[0] = st0;
    r[1] = st1;
    r[2] = 0.5 * red[2][0];
    r[3] = red[3][0];
    const unsigned long long now = globaltimer();
    r[4] = (double)(now - t0);
    r[5] = 0;
    if (la.budget_ns >= 0 && (long long)(now - t0) > la.budget_ns) {
      la.state[2] = 1;
      __threadfence();
    }
  }
  __syncthreads();  // red[][] is rewritten later
  return sqrt(st1) / fmax(sqrt(st0), 1e-12);
}

template <typename Real, bool EXACT, int CTM>  // CTM: bit 0 CTA-tile forward, bit 1 CTA-tile adjoint
__global__ void __launch_bounds__(512, 1) spgm_loop_kernel(LoopArgs la, FwdArgs<Real> fa, AdjArgs<Real> aa, CtArgs ca,
                                                           CtArgs cf) {
  constexpr bool CT = (CTM & 1) != 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int scan_sh[32];
  // sort / reduce / statistics scratch in the warp regions (no warp unit is in flight during those phases)
  double(*red)[256] = reinterpret_cast<double(*)[256]>(smem_raw);
  double(*grp_sh)[8] = reinterpret_cast<double(*)[8]>(smem_raw + 4 * 256 * sizeof(double));
  const Geo& g = fa.g;
  const int NW = blockDim.x >> 5, w = threadIdx.x >> 5, L = threadIdx.x & 31;
  // global warp index, CTA-fastest: the first units of a phase land on different SMs (small problems get one
  // warp per SM instead of a few busy SMs)
  const int gw = w * gridDim.x + blockIdx.x, TW = gridDim.x * NW;
  const int B = la.B;
  const int nfu = fa.t1 * fa.Q + (g.ntiles - fa.t1) * fa.Q2;
  const int nau = aa.t1 * aa.CH + (g.ntiles - aa.t1) * aa.CH2;
  unsigned char* wbase = smem_raw + (size_t)w * la.warp_bytes;
  const unsigned long long t0 = globaltimer();
  unsigned nbar = 0;  // grid barriers passed (grid_sync)
  int done = 0, reason = 0, k = 0;
#define LOOP_STAMP(i) \
  if (la.prof && blockIdx.x == 0 && threadIdx.x == 0) la.prof[(size_t)k * LOOP_PROF + (i)] = globaltimer() - t0
  if (loop_skip(la)) return;
  // one CTA sorts each iteration's batch into the shared records of its parity (the last CTA: CTA 0 does level 2
  // in P3); everybody reads them after the grid barriers that separate P3 from the phases that use them
  const bool sorter = blockIdx.x == gridDim.x - 1;
  if (sorter) loop_sort(la, 0, scan_sh, smem_raw);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // unit counters (a launch may have stopped between their resets)
    la.ctr[0] = 0;
    la.ctr[1] = 0;
  }
  grid_sync(la.bar, nbar);
  for (; k < la.K; ++k) {
    LOOP_STAMP(0);
    const Real* s_in = reinterpret_cast<const Real*>((k & 1) ? la.s_b : la.s_a);
    Real* s_out = reinterpret_cast<Real*>((k & 1) ? la.s_a : la.s_b);
    const size_t pbase = (size_t)(k & 1) * B;  // the records of iteration k
    // ---- forward(k) on the records sorted during iteration k-1
    // the sorting CTA first writes the next iteration's records (the other parity: last read by adjoint(k-1)); its
    // forward range is shorter by about that time (cf, ct_args kind 2; warp units are fetched dynamically anyway)
    if (sorter && k + 1 < la.K) loop_sort(la, k + 1, scan_sh, smem_raw);
    if constexpr (CT) {
      // the other phases reuse this shared memory (sort, reduce and adjoint scratch): fresh mbarriers every time
      ct_init(smem_raw);
      unsigned ph = 0;
      ct_forward<Real, EXACT, true>(fa, cf, smem_raw, s_in, la.crec + pbase, ph, false);
    } else {
      for (int u = gw; u < nfu; u = next_unit(la.ctr, TW, L))
        fwd_unit<Real, EXACT, true>(fa, u, wbase, 0, L, s_in, la.crec + pbase);
    }
    LOOP_STAMP(1);
    if (la.prof && la.prof_cta) {  // diagnostics: the whole CTA's end of the phase
      __syncthreads();
      if (threadIdx.x == 0) la.prof[(size_t)la.K * LOOP_PROF + ((size_t)k * 2) * LOOP_PROF_CTA + blockIdx.x] = globaltimer() - t0;
    }
    grid_sync(la.bar, nbar);  // B1
    LOOP_STAMP(2);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // every warp is past its forward fetches of k, adjoint fetches of k-1
      la.ctr[0] = 0;
      la.ctr[1] = 0;
    }
    if (sorter && k > 0) {  // statistics of iteration k-1 on one CTA, beside the others' reduce; its stop decision
                            // (state[2]: 2 tolerance, 1 time budget) takes effect after the next barrier
      const double change = loop_stats(la, k - 1, g.ntiles, red, grp_sh[0], t0, true);
      if (threadIdx.x == 0 && change < la.tol) la.state[2] = 2;
    }
    // ---- the forward reduce and the residual records in one phase, per channel, on the other CTAs (JC consecutive
    //      channels each): thread (seg, jj) sums the tiles of its segment in order (fwd_reduce1_kernel's sum), thread
    //      jj then the segments in order (fwd_reduce2_kernel's), y = p_f/(4pi) sum rounded to Real as stored, the
    //      residual record (resid_kernel) and |y - y_meas|^2 for the statistics (e2, parity k & 1, in la.tmp)
    if (!sorter || gridDim.x == 1) {
      const int nred = max(1, (int)gridDim.x - 1);
      const int JC = (B + nred - 1) / nred;
      const int j0 = blockIdx.x * JC, jn = min(JC, B - j0);
      double2* seg_sh = reinterpret_cast<double2*>(smem_raw);  // [nseg][JC]
      double pre = 0, pim = 0, ymr = 0, ymi = 0;
      if ((int)threadIdx.x < jn) {  // the finishing threads' record loads go first
        const double2 pf = la.yrec[2 * (pbase + j0 + threadIdx.x)], ym = la.yrec[2 * (pbase + j0 + threadIdx.x) + 1];
        pre = pf.x;
        pim = pf.y;
        ymr = ym.x;
        ymi = ym.y;
      }
      // The CTA's partials [tiles][jn] go through shared memory in chunks of la.stage_tiles tiles (asynchronous
      // copies, so the loads in flight are not bounded by registers; BASELINE Medium: one chunk); thread (seg, jj)
      // adds its segment's tiles of the chunk in order to its running sum, kept in seg_sh between chunks.
      R2<Real>* stage = reinterpret_cast<R2<Real>*>(seg_sh + (size_t)la.nseg * JC);
      const int cap = la.stage_tiles;
      const int nitems = la.nseg * jn;
      if (cap > 0) {
        const R2<Real>* src = reinterpret_cast<const R2<Real>*>(fa.part) + j0;
        for (int xa = 0; xa < g.ntiles; xa += cap) {
          const int xb = min(g.ntiles, xa + cap);
          const int total = (xb - xa) * jn;
          for (int it = threadIdx.x; it < total; it += blockDim.x) {
            const int x = (int)((unsigned)it / (unsigned)jn), jj = it - x * jn;
            const unsigned d = (unsigned)__cvta_generic_to_shared(stage + it);
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src + (size_t)(xa + x) * B + jj),
                         "n"((int)sizeof(R2<Real>))
                         : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
          asm volatile("cp.async.wait_all;" ::: "memory");
          __syncthreads();
          if (xa == 0) LOOP_STAMP(3);
          for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
            const int seg = (int)((unsigned)it / (unsigned)jn), jj = it - seg * jn;
            // (tiles * segments < 2^31: the same quotients as the 64-bit form of fwd_reduce1_kernel)
            const int x0 = (int)((unsigned)(g.ntiles * seg) / (unsigned)la.nseg);
            const int x1 = (int)((unsigned)(g.ntiles * (seg + 1)) / (unsigned)la.nseg);
            const int lo = max(x0, xa), hi = min(x1, xb);
            if (lo >= hi && !(xa == 0 && x0 >= x1)) continue;
            double sr = 0, si = 0;
            if (lo > x0) {
              const double2 acc = seg_sh[seg * JC + jj];
              sr = acc.x;
              si = acc.y;
            }
#pragma unroll 4
            for (int x = lo; x < hi; ++x) {
              const R2<Real> v = stage[(x - xa) * jn + jj];
              sr += (double)v.x;
              si += (double)v.y;
            }
            seg_sh[seg * JC + jj] = make_double2(sr, si);
          }
          __syncthreads();
        }
      } else {
        LOOP_STAMP(3);
        for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
          const int seg = it / jn, jj = it - seg * jn;
          const int x0 = (int)((unsigned)(g.ntiles * seg) / (unsigned)la.nseg);
          const int x1 = (int)((unsigned)(g.ntiles * (seg + 1)) / (unsigned)la.nseg);
          const R2<Real>* src = reinterpret_cast<const R2<Real>*>(fa.part) + j0 + jj;
          double sr = 0, si = 0;
#pragma unroll 8
          for (int x = x0; x < x1; ++x) {
            const R2<Real> v = src[(size_t)x * B];
            sr += (double)v.x;
            si += (double)v.y;
          }
          seg_sh[seg * JC + jj] = make_double2(sr, si);
        }
      }
      __syncthreads();
      LOOP_STAMP(4);
      if ((int)threadIdx.x < jn) {
        const int j = j0 + threadIdx.x;
        double sr = 0, si = 0;
        for (int sgi = 0; sgi < la.nseg; ++sgi) {
          const double2 v = seg_sh[sgi * JC + threadIdx.x];
          sr += v.x;
          si += v.y;
        }
        const double pr = pre / (4.0 * PI), pi_ = pim / (4.0 * PI);  // (the quotients the per-launch kernels form)
        const Real yr = (Real)(pr * sr - pi_ * si), yi = (Real)(pr * si + pi_ * sr);
        double rr = (double)yr, ri = (double)yi;
        rr -= ymr;
        ri -= ymi;
        const double qr = pre / (4.0 * PI), qi = -pim / (4.0 * PI);
        R2<Real> wv;
        wv.x = (Real)(qr * rr - qi * ri);
        wv.y = (Real)(qr * ri + qi * rr);
        const_cast<R2<Real>*>(aa.wrec)[j] = wv;
        reinterpret_cast<double*>(la.tmp)[(size_t)(k & 1) * B + j] = rr * rr + ri * ri;
      }
    }
    LOOP_STAMP(5);
    grid_sync(la.bar, nbar);  // B3
    LOOP_STAMP(6);
    if (k > 0) {  // iteration k-1 was the last (every CTA reads the same flag): k iterations ran
      const int stop = *(volatile int*)(la.state + 2);
      if (stop) {
        done = k;
        reason = stop == 2 ? 1 : 2;
        break;
      }
    }
    // ---- adjoint(k) + prox
    if constexpr ((CTM & 2) != 0) {
      ct_init(smem_raw);  // the sort of P3 used this shared memory
      unsigned ph = 0;
      ct_adjoint<Real, true, EXACT, true>(aa, ca, smem_raw, s_in, s_out, la.crec + pbase,
                                          reinterpret_cast<Real*>(la.ctpart), la.ctpmax, ph, false);
    } else {
      for (int u = gw; u < nau; u = next_unit(la.ctr + 1, TW, L))
        adj_unit<Real, true, EXACT, true>(aa, u, wbase, L, s_in, s_out, la.crec + pbase);
    }
    LOOP_STAMP(7);
    if (la.prof && la.prof_cta) {  // diagnostics: the whole CTA's end of the phase
      __syncthreads();
      if (threadIdx.x == 0) la.prof[(size_t)la.K * LOOP_PROF + ((size_t)k * 2 + 1) * LOOP_PROF_CTA + blockIdx.x] = globaltimer() - t0;
      if (threadIdx.x == 0 && k == 0) {  // the SM of this CTA, in a row after the stamps
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        la.prof[(size_t)la.K * LOOP_PROF + (size_t)la.K * 2 * LOOP_PROF_CTA + blockIdx.x] = smid;
      }
    }
    grid_sync(la.bar, nbar);  // B4
    LOOP_STAMP(8);
    done = k + 1;
  }
  if (k == la.K && blockIdx.x == 0) {  // every iteration ran: the statistics of the last one
    const double change = loop_stats(la, la.K - 1, g.ntiles, red, grp_sh[0], t0, true);
    if (change < la.tol) reason = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (reason == 0 && la.state[2] == 1) reason = 2;  // the budget ran out on the last iteration of the launch
    la.state[0] = done;
    la.state[1] = reason;
  }
  loop_fold<Real>(la, done, (long long)g.nx * g.ny * g.nzs);
}
#undef LOOP_STAMP


// ------------------------------------------------------------------ persistent loop for tiny problems
//
// BASELINE Small (|B| = 32, N = 2048) has 65,536 entries per operator application: every warp unit of the
// flat kernels is then a chain of start-up latencies (~10 us) rather than work. tiny_loop_kernel runs the
// SPGM iteration for such problems (|B|·N <= TINY_MAX_ENTRIES) with one thread per voxel and the entries
// evaluated straight from the geometry in fp64 (distances, phase in revolutions reduced exactly, table
// cis), between three grid barriers per iteration:
//   PA  items (channel group of JC, block of 256 voxels): each thread forms A[m_j, n]·s_n for its voxel and
//       the block sums them in a fixed order -> part[vb][j]
//   PB  per channel: y_j = p_f/(4π)·Σ_vb part[vb][j] (fixed order), residual record w_j = conj(p_f)/(4π)·(y_j −
//       y_meas[m_j]) and ½|y_j − y_meas|² per 256-channel group
//   PC  items (voxel block, channel chunk): thread-per-voxel Σ_j conj(A)·w_j -> gpart; the last chunk of a
//       voxel block to finish sums the chunks in order, applies s − η/B·g and the complex soft threshold,
//       and writes the block's termination statistics
//   PD  every CTA reduces the statistics in a fixed order, records them and tests the tolerance
// The arithmetic differs from the flat kernels' (per-voxel fp64 entries, different summation trees) but is
// fixed for a given plan, batch and iterate: results are deterministic, and agree with the reference to the
// c128 tolerance (tests/test_gpu_loop.py).
constexpr long long TINY_MAX_ENTRIES = 1LL << 20;  // |B| x slab voxels
constexpr int TINY_JC = 8;                         // channels per PA item, at most

struct TinyArgs {
  const double* ant;   // [A][3] antenna positions (tx then rx)
  const double* kd;    // f / c
  double corner[3], sp[3];
  int nx, ny, nzs, zb, T, R;
  int nvb, jc, cc;     // voxel blocks of 256, channels per PA item, channel chunks per PC voxel block
  int chunk_max;       // largest PC channel chunk
  double2* part;       // [nvb][B]
  double* e2;          // [B] |y_j - y_meas|^2
  double2* gpart;      // [cc][nvb][256]
  int* vbcnt;          // [nvb] arrival counters (zero between iterations)
  double* stat_part;   // [nvb][4]
};

// e^{-j 2π kd (dT + dR)} / (dT dR) for voxel centre (x, y, z) and channel (t, r, kd), in fp64
__device__ __forceinline__ double2 tiny_entry(const TinyArgs& ta, double x, double y, double z, int t, int r,
                                             double kd) {
  const double* a = ta.ant + 3 * t;
  const double* b = ta.ant + 3 * (ta.T + r);
  const double qT = (x - a[0]) * (x - a[0]) + (y - a[1]) * (y - a[1]) + (z - a[2]) * (z - a[2]);
  const double qR = (x - b[0]) * (x - b[0]) + (y - b[1]) * (y - b[1]) + (z - b[2]) * (z - b[2]);
  const double iT = rsqrt(qT), iR = rsqrt(qR);  // 1/d within 1 ulp; d = q/sqrt(q) within 2 ulp
  const double rev = kd * fma(qT, iT, qR * iR);
  double s, c;
  cis_rev(rev - rint(rev), s, c);
  const double amp = iT * iR;
  return make_double2(c * amp, -s * amp);
}

__device__ __forceinline__ void tiny_voxel(const TinyArgs& ta, int n, double& x, double& y, double& z) {
  const int ix = n % ta.nx, q = n / ta.nx, iy = q % ta.ny, iz = q / ta.ny + ta.zb;
  x = ta.corner[0] + ix * ta.sp[0];
  y = ta.corner[1] + iy * ta.sp[1];
  z = ta.corner[2] + iz * ta.sp[2];
}

// fixed-order sum over the 256 threads of a CTA of JC complex values: warp trees, then warps in order
__device__ __forceinline__ void tiny_block_sum(double2* v, int jc, double2 (*sh)[TINY_JC]) {
  const int L = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < TINY_JC; ++q) {
    if (q >= jc) break;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[q].x += __shfl_xor_sync(FULL, v[q].x, o);
      v[q].y += __shfl_xor_sync(FULL, v[q].y, o);
    }
    if (L == 0) sh[w][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < jc) {
    double2 t = make_double2(0, 0);
    for (int i = 0; i < 8; ++i) {
      t.x += sh[i][threadIdx.x].x;
      t.y += sh[i][threadIdx.x].y;
    }
    v[0] = t;  // thread q < jc holds the sum of channel q
  }
  __syncthreads();
}

template <typename Real>
__global__ void __launch_bounds__(256, 1) tiny_loop_kernel(LoopArgs la, TinyArgs ta) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double2 bsum[8][TINY_JC];
  __shared__ double red[4][256];
  __shared__ int last_sh;
  double2* wsm = reinterpret_cast<double2*>(smem_raw);  // [chunk] residual records of the item's channel chunk
  int4* csm = reinterpret_cast<int4*>(smem_raw + (size_t)ta.chunk_max * sizeof(double2));  // [chunk] channels
  const int B = la.B, nvb = ta.nvb, jc = ta.jc, cc = ta.cc;
  const long long nvox = (long long)ta.nx * ta.ny * ta.nzs;
  const Real* ym = reinterpret_cast<const Real*>(la.ymeas);
  const unsigned long long t0 = globaltimer();
  unsigned nbar = 0;  // grid barriers passed (grid_sync)
  int done = 0, reason = 0;
  if (loop_skip(la)) return;
#define TINY_STAMP(i) \
  if (la.prof && blockIdx.x == 0 && threadIdx.x == 0) la.prof[(size_t)k * LOOP_PROF + (i)] = globaltimer() - t0
  for (int k = 0; k < la.K; ++k) {
    TINY_STAMP(0);
    const Real* s_in = reinterpret_cast<const Real*>((k & 1) ? la.s_b : la.s_a);
    Real* s_out = reinterpret_cast<Real*>((k & 1) ? la.s_a : la.s_b);
    // ---- PA: forward partials per (channel group, voxel block)
    const int ngrp = (B + jc - 1) / jc;
    for (int item = blockIdx.x; item < ngrp * nvb; item += gridDim.x) {
      const int jg = item / nvb, vb = item - jg * nvb;
      const int n = vb * 256 + threadIdx.x;
      double2 v[TINY_JC];
      double sr = 0, si = 0, x = 0, y = 0, z = 0;
      if (n < nvox) {
        sr = (double)s_in[2 * (size_t)n];
        si = (double)s_in[2 * (size_t)n + 1];
        tiny_voxel(ta, n, x, y, z);
      }
#pragma unroll
      for (int q = 0; q < TINY_JC; ++q) {
        v[q] = make_double2(0, 0);
        const int j = jg * jc + q;
        if (q < jc && j < B && n < nvox) {
          const int m = loop_index(la, k, j);
          const int f = m / (ta.T * ta.R), rem = m - f * ta.T * ta.R, t = rem / ta.R, r = rem - t * ta.R;
          const double2 e = tiny_entry(ta, x, y, z, t, r, ta.kd[f]);
          v[q] = make_double2(e.x * sr - e.y * si, e.x * si + e.y * sr);
        }
      }
      tiny_block_sum(v, jc, bsum);
      const int j = jg * jc + threadIdx.x;
      if (threadIdx.x < jc && j < B) ta.part[(size_t)vb * B + j] = v[0];
    }
    TINY_STAMP(1);
    grid_sync(la.bar, nbar);
    TINY_STAMP(2);
    if (k > 0 && *(volatile int*)(la.state + 2)) {
      reason = 2;
      break;
    }
    // ---- PC: per (voxel block, channel chunk): the chunk's channel sums and residual records (recomputed by
    // each of its voxel blocks from the same partials in the same order, so no barrier is needed before the
    // adjoint; the vb = 0 item keeps ½|r_j|² for the statistics), the adjoint partial of the block over the
    // chunk -> gpart; the last chunk of a voxel block to finish sums the chunks in order and applies the prox
    for (int item = blockIdx.x; item < nvb * cc; item += gridDim.x) {
      const int vb = item / cc, c = item - vb * cc;
      const int n = vb * 256 + threadIdx.x;
      const int j0 = (int)(((long long)B * c) / cc), j1 = (int)(((long long)B * (c + 1)) / cc);
      for (int j = j0 + threadIdx.x; j < j1; j += 256) {
        const int m = loop_index(la, k, j);
        const int f = m / (ta.T * ta.R), rem = m - f * ta.T * ta.R, t = rem / ta.R, r = rem - t * ta.R;
        double sr = 0, si = 0;
        for (int q = 0; q < nvb; ++q) {
          const double2 pp = __ldcg(ta.part + (size_t)q * B + j);
          sr += pp.x;
          si += pp.y;
        }
        const double pr = la.pulse[2 * f] / (4.0 * PI), pim = la.pulse[2 * f + 1] / (4.0 * PI);
        const Real yr = (Real)(pr * sr - pim * si), yi = (Real)(pr * si + pim * sr);
        const double rr = (double)yr - (double)ym[2 * (size_t)m], ri = (double)yi - (double)ym[2 * (size_t)m + 1];
        wsm[j - j0] = make_double2(pr * rr + pim * ri, pr * ri - pim * rr);  // conj(p)/(4π)·r
        csm[j - j0] = make_int4(f, t, r, m);
        if (vb == 0) ta.e2[j] = rr * rr + ri * ri;
      }
      __syncthreads();
      double gr = 0, gi = 0;
      if (n < nvox) {
        double x, y, z;
        tiny_voxel(ta, n, x, y, z);
        for (int j = 0; j < j1 - j0; ++j) {
          const int4 q = csm[j];
          const double2 e = tiny_entry(ta, x, y, z, q.y, q.z, ta.kd[q.x]);
          const double2 wv = wsm[j];
          gr += e.x * wv.x + e.y * wv.y;  // conj(e)·w
          gi += e.x * wv.y - e.y * wv.x;
        }
      }
      ta.gpart[((size_t)c * nvb + vb) * 256 + threadIdx.x] = make_double2(gr, gi);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) last_sh = atomicAdd(ta.vbcnt + vb, 1) == cc - 1;
      __syncthreads();
      if (!last_sh) continue;
      __threadfence();
      double st0 = 0, st1 = 0, st3 = 0;
      if (n < nvox) {
        gr = gi = 0;
        for (int q = 0; q < cc; ++q) {
          const double2 pp = __ldcg(ta.gpart + ((size_t)q * nvb + vb) * 256 + threadIdx.x);
          gr += pp.x;
          gi += pp.y;
        }
        const Real s_r = s_in[2 * (size_t)n], s_i = s_in[2 * (size_t)n + 1];
        const Real ur = s_r - (Real)la.eta_over_b * (Real)gr, ui = s_i - (Real)la.eta_over_b * (Real)gi;
        const Real mag = hypot(ur, ui);
        const Real al = (Real)la.alpha;
        const Real sc = mag > al ? (mag - al) / mag : Real(0);
        const Real o_r = ur * sc, o_i = ui * sc;
        s_out[2 * (size_t)n] = o_r;
        s_out[2 * (size_t)n + 1] = o_i;
        const double m0 = hypot((double)s_r, (double)s_i), m1 = hypot((double)o_r, (double)o_i);
        st0 = m0 * m0;
        st1 = (m1 - m0) * (m1 - m0);
        st3 = m1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        st0 += __shfl_xor_sync(FULL, st0, o);
        st1 += __shfl_xor_sync(FULL, st1, o);
        st3 += __shfl_xor_sync(FULL, st3, o);
      }
      if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = st0;
        red[1][threadIdx.x >> 5] = st1;
        red[3][threadIdx.x >> 5] = st3;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double a0 = 0, a1 = 0, a3 = 0;
        for (int i = 0; i < 8; ++i) {
          a0 += red[0][i];
          a1 += red[1][i];
          a3 += red[3][i];
        }
        ta.stat_part[(size_t)vb * 4 + 0] = a0;
        ta.stat_part[(size_t)vb * 4 + 1] = a1;
        ta.stat_part[(size_t)vb * 4 + 2] = 0;
        ta.stat_part[(size_t)vb * 4 + 3] = a3;
        ta.vbcnt[vb] = 0;
      }
      __syncthreads();
    }
    TINY_STAMP(3);
    grid_sync(la.bar, nbar);
    TINY_STAMP(4);
    // ---- PD: statistics (fixed order, every CTA), record, termination
    if (nvb <= 256 && B <= 1024) {  // one warp: lane-strided sums, then a shuffle tree (no block barriers)
      if (threadIdx.x < 32) {
        double acc[4] = {0, 0, 0, 0};
        for (int i = threadIdx.x; i < nvb; i += 32) {
          acc[0] += __ldcg(ta.stat_part + (size_t)i * 4 + 0);
          acc[1] += __ldcg(ta.stat_part + (size_t)i * 4 + 1);
          acc[3] += __ldcg(ta.stat_part + (size_t)i * 4 + 3);
        }
        for (int i = threadIdx.x; i < B; i += 32) acc[2] += __ldcg(ta.e2 + i);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(FULL, acc[q], o);
          if (threadIdx.x == 0) red[q][0] = acc[q];
        }
      }
      __syncthreads();
    } else {
      double acc[4] = {0, 0, 0, 0};
      for (int i = threadIdx.x; i < nvb; i += 256) {
        acc[0] += ta.stat_part[(size_t)i * 4 + 0];
        acc[1] += ta.stat_part[(size_t)i * 4 + 1];
        acc[3] += ta.stat_part[(size_t)i * 4 + 3];
      }
      for (int i = threadIdx.x; i < B; i += 256) acc[2] += ta.e2[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = acc[q];
      __syncthreads();
      for (int sh = 128; sh > 0; sh >>= 1) {
        if (threadIdx.x < sh)
#pragma unroll
          for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + sh];
        __syncthreads();
      }
    }
    const double st0 = red[0][0], st1 = red[1][0];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double* r = la.rec + (size_t)k * LOOP_REC;
      r[0] = st0;
      r[1] = st1;
      r[2] = 0.5 * red[2][0];
      r[3] = red[3][0];
      const unsigned long long now = globaltimer();
      r[4] = (double)(now - t0);
      r[5] = 0;
      if (la.budget_ns >= 0 && (long long)(now - t0) > la.budget_ns) {
        la.state[2] = 1;
        __threadfence();
      }
    }
    done = k + 1;
    TINY_STAMP(5);
    const double change = sqrt(st1) / fmax(sqrt(st0), 1e-12);
    if (change < la.tol) {
      reason = 1;
      break;
    }
    __syncthreads();
  }
#undef TINY_STAMP
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (reason == 0 && la.state[2]) reason = 2;
    la.state[0] = done;
    la.state[1] = reason;
  }
  loop_fold<Real>(la, done, nvox);
}
template __global__ void tiny_loop_kernel<float>(LoopArgs, TinyArgs);
template __global__ void tiny_loop_kernel<double>(LoopArgs, TinyArgs);

}  // namespace

// ====================================================================== plan
struct nf_plan {
  Geo g;
  int dtype;
  int M;
  int max_batch;
  int B = 0;
  double c;
  int64_t nvox;
  int fwd_gridx;
  int fwd_nseg;        // level-1 segments of the forward reduce: a function of the plan only (bit-exact subsets)
  int fwd_chunk;
  size_t tmp_elems = 0;  // d_tmp capacity (double2)
  int adj_ch_cap;
  bool exact = true;  // explicit phase reduction (false when |x| <= EXACT_FREE_REV is guaranteed)
  double phase_bound_rev = 0;
  long long fwd_target = 148LL * 16 * 4;  // warp work units per forward launch (env NFGPU_FWD_TARGET)
  long long adj_target = 148LL * 16 * 4;  // warp work units per adjoint launch (set with chunk_order; env NFGPU_ADJ_TARGET)
  long long struct_target = 148LL * 3 * 4;  // blocks per structured launch (env NFGPU_STRUCT_TARGET)
  int min_chunk = 64;                       // fewest channels per flat forward unit (env NFGPU_MIN_CHUNK)
  int chunk_order = 0;                      // flat work-unit order (unit_coords / chunk_bound)
  bool tail_split = true;                   // tile-major launches end on shorter units (unit_map; env NFGPU_TAIL=0)
  int tail_factor = 4;                      // ... tail_factor x more chunks per tail tile (env NFGPU_TAIL_FACTOR)
  // wave_fit: bit 0 forward, bit 1 adjoint. Per-launch kernels: the adjoint only (Medium step 119.5 -> 116.0 us;
  // the hardware's CTA scheduler already balances the forward); the persistent loop, whose warps fetch units
  // themselves: both (Medium loop 126.4 -> 121.5 us with the forward). Env NFGPU_WAVE_FIT / NFGPU_LOOP_WAVE_FIT.
  int wave_fit = 2;
  int loop_wave_fit = 3;
  double ct_cost_fwd = 80, ct_cost_adj = 150;  // fixed cost of a CTA-tile piece, in (tile, channel) pairs (ct_args;
                                               // env NFGPU_CT_COST_FWD / NFGPU_CT_COST_ADJ, 0: equal ranges)
  struct CtCache {
    int span = -1, G = 0;
    double cost = -1, disc = -1;
    CtArgs args;
  };
  mutable CtCache ct_cache[3];
  double loop_sort_disc = 12.0;  // % of an equal forward share the loop's sorting CTA is spared (NFGPU_SORT_DISC)
  int fit_min_waves = 1;  // env NFGPU_FIT_MIN_WAVES
  double tail_waves = 1.0;                  // ... for about this many waves of warp slots (env NFGPU_TAIL_WAVES)
  double taper = 0.375;                     // chunk-major adjoint taper h: last chunk 1 − 2h of the first (env NFGPU_TAPER)
  double fwd_taper = 0.475;                 // ... forward (1/8 Large slab 0.3552 -> 0.3516 ms; env NFGPU_FWD_TAPER)
  int adj_min_chunk = 128;                  // ... per flat adjoint unit: its chunk combine favours fewer, longer
                                            // chunks (Medium |B| = 512: 80.9 -> 72.7 us; env NFGPU_ADJ_MIN_CHUNK)
  size_t dev_bytes = 0;
  int64_t launches = 0;
  int KS, ksblocks;
  KeyMap km;     // batch order of the warp-unit kernels
  KeyMap km_rx;  // ... of the CTA-tile kernels (rx-major; ct_rxmajor)
  bool rxmajor = false;  // the staged flat batch is in rx-major order
  // device
  double* d_ant = nullptr;
  double* d_kd = nullptr;
  void* d_kf = nullptr;
  double* d_pulse = nullptr;
  void* d_tab = nullptr;
  double* d_D0 = nullptr;
  int* d_pos_of_key = nullptr;
  int* d_cnt = nullptr;
  int* d_sm = nullptr;
  int* d_spos = nullptr;
  ChanRec* d_crec = nullptr;
  int* d_sf = nullptr;
  void* d_wrec = nullptr;
  double* d_dpart = nullptr;
  void* d_part = nullptr;
  double2* d_tmp = nullptr;
  void* d_gpart = nullptr;
  int* d_tilecnt = nullptr;
  double* d_stat_part = nullptr;
  unsigned long long* d_iter = nullptr;
  // structured (Cartesian) batch: sorted frequency / tx / rx index lists at fixed offsets [F | T | R]
  bool structured = false;
  int snf = 0, snt = 0, snr = 0;
  int* d_struct = nullptr;
  // tensor-core structured adjoint (c64): B images [batch frequency][K chunk][hi|lo][npad][16]
  bool use_tc = false;
  bool tc_force = false;  // NFGPU_TC=2: tensor-core kernels whenever eligible (tests)
  bool use_pdl = true;    // programmatic dependent launch of the SPGM step kernels (env NFGPU_PDL=0 disables)
  bool tc_fwd = false;    // NFGPU_TC_FWD=1: route structured forwards to the tcgen05 forward
  float* d_bimg = nullptr;
  // tensor-core structured forward: per-(half tile, channel) partials, allocated on first use
  float2* d_tcpart = nullptr;
  size_t tcpart_elems = 0;
  // peer all-reduce of the forward partials (nf_comm_*): own buffer = receive slots
  // [2][world][comm_cap] double2, then flags [world][comm_nblk] u64; peers mapped by CUDA IPC
  int comm_world = 0, comm_rank = -1, comm_cap = 0, comm_nblk = 0;
  bool comm_connected = false;
  void* comm_buf = nullptr;
  void* comm_peer[PEER_MAX] = {};
  unsigned long long* d_epoch = nullptr;
  int* d_comm_err = nullptr;
  unsigned* d_loopbar = nullptr;  // persistent SPGM loop: grid barrier arrival counter (zeroed before every launch), unit counters
  int loop_threads = 0;           // ... CTA size chosen on first use (0: not yet)
  unsigned long long* d_loop_prof = nullptr;  // ... phase time stamps (NFGPU_LOOP_PROFILE)
  void* d_loop_priv = nullptr;  // spgm_loop_kernel: sorted records of two iterations
  size_t loop_priv_bytes = 0;
  void* d_tiny = nullptr;  // tiny_loop_kernel scratch: part, wch, ch, gpart, vbcnt, stat_part
  size_t tiny_bytes = 0;
  size_t loop_prof_elems = 0;
  const int* loop_prev = nullptr;  // nf_spgm_loop_chained: the previous launch's state (LoopArgs::prev_state)
  int loop_fold = 0;               // ... and LoopArgs::fold
  int nsm = 148;             // SMs of the plan's device: CTAs of the CTA-tile forward and the persistent loop
  int ct_mode = 1;           // CTA-tile flat forward (use_ct): 0 off, 1 when the work is large enough, 2 whenever
                             // the layout fits (tests); env NFGPU_CT
  long long ct_min_pairs = 1024;  // ... fewest (tile, channel) pairs per CTA (env NFGPU_CT_MIN)
  int ct_adj = 1;                 // CTA-tile adjoint too (when use_ct holds for the batch; env NFGPU_CT_ADJ)
  int ct_rx = 1;                  // rx-major order for batches on the CTA-tile kernels (env NFGPU_CT_RXMAJOR)
  void* d_ctpart = nullptr;       // ... its parked piece sums
  size_t ctpart_bytes = 0;
  bool comm_active = false;  // inside nf_forward_allreduce
  bool comm_fused = false;   // ... and the flat forward's last reduce already did the all-reduce
};

namespace {

// launch with programmatic dependent launch when enabled (the kernel must begin with pdl_wait())
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename T>
int dalloc(nf_plan* p, T** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc((void**)ptr, bytes);
  if (e != cudaSuccess)
    return fail(NF_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  p->dev_bytes += bytes;
  return NF_OK;
}

// Set a kernel's dynamic shared-memory limit (and the carveout) only when a launch needs more than was set
// before on the current device (each cudaFuncSetAttribute call costs host time on every per-call launch).
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_attr_smem;
cudaError_t ensure_smem(const void* kern, size_t bytes, bool carveout = false) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& cur = g_attr_smem[{kern, dev}];
  if ((int)bytes <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && carveout)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) cur = (int)bytes;
  return e;
}

void free_plan(nf_plan* p) {
  if (!p) return;
  void* ptrs[] = {p->d_ant,  p->d_kd,   p->d_kf,    p->d_pulse, p->d_tab,  p->d_D0,      p->d_pos_of_key,
                  p->d_cnt,  p->d_sm,   p->d_spos,  p->d_crec,  p->d_sf, p->d_wrec, p->d_dpart,   p->d_part,
                  p->d_tmp,  p->d_gpart, p->d_tilecnt, p->d_stat_part, p->d_iter, p->d_struct, p->d_bimg, p->d_tcpart};
  for (void* q : ptrs) cudaFree(q);
  for (int q = 0; q < p->comm_world; ++q)
    if (q != p->comm_rank && p->comm_peer[q]) cudaIpcCloseMemHandle(p->comm_peer[q]);
  cudaFree(p->comm_buf);
  cudaFree(p->d_loopbar);
  cudaFree(p->d_loop_prof);
  cudaFree(p->d_tiny);
  cudaFree(p->d_loop_priv);
  cudaFree(p->d_ctpart);
  cudaFree(p->d_epoch);
  cudaFree(p->d_comm_err);
  delete p;
}

// level-1 segments of the two-level forward reduce over `rows` partial rows: ~sqrt(rows), so both levels
// have short serial sums; a function of the row count only
int reduce_segments(int rows) {
  return std::max(1, std::min(rows, (int)std::ceil(std::sqrt((double)rows))));
}

size_t real_size(const nf_plan* p) { return p->dtype == NF_C64 ? sizeof(float) : sizeof(double); }

size_t fwd_smem(const nf_plan* p) {
  const int Tg = p->g.Tg;
  if (p->dtype == NF_C64) return FWD_WARPS * fwd_warp_bytes<float>(Tg, p->g.A);
  return FWD_WARPS * fwd_warp_bytes<double>(Tg, p->g.A);
}
size_t adj_smem(const nf_plan* p) {
  return ADJ_WARPS * (p->dtype == NF_C64 ? warp_smem_bytes<float>(p->g.Tg, p->g.A)
                                          : warp_smem_bytes<double>(p->g.Tg, p->g.A));
}

// Tapered chunk-major units pay off only with several waves of units: with fewer, the tapered
// first chunk (1.6x the mean at 4 chunks) is the critical path (Medium: 135 -> 156 us per step).
int unit_order(const nf_plan* p, long long units) {
  return p->chunk_order && units >= 2LL * 148 * 16 ? 1 : 0;
}

// Tile-major split tail (unit_map): the last tiles take 4x as many (so 4x shorter) chunks, enough of them for
// about one wave of warp slots, so the launch does not end on a wave of long units. cmax bounds the chunk count.
void tail_split(const nf_plan* p, int order, int C, long long cmax, int& t1, int& C2) {
  t1 = p->g.ntiles;
  C2 = C;
  if (order != 0 || !p->tail_split) return;
  const long long c2 = std::min<long long>((long long)p->tail_factor * C, cmax);
  if (c2 <= C) return;
  const long long slots = (long long)(148.0 * 16 * p->tail_waves);
  const long long ntail = std::min<long long>(p->g.ntiles, (slots + c2 - 1) / c2);
  t1 = p->g.ntiles - (int)ntail;
  C2 = (int)c2;
}

// Wave fit for tile-major launches without a split tail (Medium-sized problems, whose equal units leave the last
// wave partly empty: BASELINE Medium's 4096 forward units fill 1.73 waves of the 2368 warp slots): tiles
// [0, t1) take C chunks and tiles [t1, ntiles) C + 1, so the unit count is exactly k waves. cmax bounds the
// chunk count (channels per tile for the forward, the partial-buffer cap for the adjoint).
void wave_fit(const nf_plan* p, int order, int cmax, int& C, int& t1, int& C2) {
  if (order != 0 || t1 != p->g.ntiles || C2 != C) return;  // chunk-major or already split
  const long long slots = 148LL * 16, nt = p->g.ntiles, units = nt * C;
  if (units < slots / 2 || units > 4 * slots) return;
  const long long target = std::max<long long>((units + slots - 1) / slots, p->fit_min_waves) * slots;
  const long long c = target / nt;
  if (c < 1 || c + 1 > cmax) return;
  t1 = (int)(nt * (c + 1) - target);
  C = (int)c;
  C2 = (int)c + 1;
}

// Chunks per tile: enough (tile, chunk) warp units for the target, with at least min_chunk channels per
// chunk -- unless that leaves less than a quarter wave of units (tiny problems such as BASELINE Small: 8 tiles,
// 32 channels), where chunks go down to SMALL_CHUNK channels to put more warps on the latency-bound work.
#ifndef NFGPU_SMALL_CHUNK
#define NFGPU_SMALL_CHUNK 4
#endif
constexpr int SMALL_CHUNK = NFGPU_SMALL_CHUNK;
long long chunks_for(const nf_plan* p, long long target, int n, int min_chunk) {
  const long long slots = 148LL * 16;
  long long q = (target + p->g.ntiles - 1) / p->g.ntiles;
  long long cap = std::max(1, n / min_chunk);
  if ((long long)p->g.ntiles * cap < slots / 4)
    cap = std::min<long long>((slots + p->g.ntiles - 1) / p->g.ntiles, std::max(1, n / SMALL_CHUNK));
  return std::max(1LL, std::min(q, cap));
}

int channel_splits(const nf_plan* p, int span) { return (int)chunks_for(p, p->fwd_target, span, p->min_chunk); }

int adjoint_chunks(const nf_plan* p) {
  return (int)std::min<long long>(chunks_for(p, p->adj_target, p->B, p->adj_min_chunk), p->adj_ch_cap);
}

size_t comm_recv_bytes(const nf_plan* p) { return (size_t)2 * p->comm_world * p->comm_cap * sizeof(double2); }

PeerArgs peer_args(const nf_plan* p, int blk_base, const void* tmp, void* y) {
  PeerArgs pa = {};
  pa.world = p->comm_world;
  pa.rank0 = p->comm_rank;
  pa.cap = p->comm_cap;
  pa.nblk_cap = p->comm_nblk;
  pa.blk_base = blk_base;
  for (int q = 0; q < p->comm_world; ++q) {
    char* base = (char*)p->comm_peer[q];
    pa.recv[q] = (double2*)base;
    pa.flag[q] = (unsigned long long*)(base + comm_recv_bytes(p));
  }
  pa.tmp[0] = (const double2*)tmp;
  pa.y[0] = y;
  pa.epoch[0] = p->d_epoch;
  pa.err = p->d_comm_err;
  return pa;
}

// Level 2 of the forward reduce: plain (scatter to y) or, inside nf_forward_allreduce on a flat batch
// (`fuse`), fused with the peer all-reduce across the plan's voxel-slab ranks (fwd_reduce2_peer_kernel).
template <typename Real>
int launch_reduce2(nf_plan* p, int span, int nseg, int w0, void* y, cudaStream_t st, bool pdl, bool fuse = false) {
  const int nblk = (span + 255) / 256;
  if (!(p->comm_active && fuse)) {
    CUDA_TRY(launch_k(pdl, fwd_reduce2_kernel<Real>, dim3(nblk), dim3(256), 0, st, (const double2*)p->d_tmp, span,
                      nseg, w0, (const int*)p->d_sf, (const int*)p->d_spos, (const double*)p->d_pulse, (Real*)y));
    return NF_OK;
  }
  if (w0 % 256 || w0 / 256 + nblk > p->comm_nblk) return fail(NF_ERR_STATE, "peer all-reduce: unaligned window");
  const PeerArgs pa = peer_args(p, w0 / 256, p->d_tmp, y);
  CUDA_TRY(launch_k(pdl, fwd_reduce2_peer_kernel<Real, false>, dim3(nblk, 1), dim3(256), 0, st, pa, span, nseg, w0,
                    (const int*)p->d_sf, (const int*)p->d_spos, (const double*)p->d_pulse));
  p->comm_fused = true;
  return NF_OK;
}

// CTA-tile forward (ct_forward) for a flat window of n channels: the whole per-tile table fits twice in shared
// memory and every CTA gets at least ct_min_pairs (tile, channel) pairs (at least one with NFGPU_CT=2)
bool use_ct(const nf_plan* p, long long n) {
  if (p->ct_mode == 0 || p->structured || n < 1) return false;
  // (the margin keeps room for the persistent loop's static shared memory, so the loop runs what nf_forward and
  // nf_adjoint_prox run: same bits)
  const size_t bytes = p->dtype == NF_C64 ? CtLayout<float>(p->g.A).bytes : CtLayout<double>(p->g.A).bytes;
  if (bytes > 232448 - 4096) return false;
  if ((long long)p->g.ntiles * n < p->nsm || (long long)p->g.ntiles * n > INT32_MAX || p->nsm > CT_GMAX) return false;
  return p->ct_mode == 2 || (long long)p->g.ntiles * n >= p->ct_min_pairs * p->nsm;
}
// ... and the CTA-tile adjoint (ct_adjoint) for a flat batch of B channels: a tile's pieces fit the chunk-partial
// buffer (adj_epilogue), and the parked piece sums are allocated (pmax per CTA)
bool use_ct_adj(const nf_plan* p, long long B) {
  if (!p->ct_adj || !use_ct(p, B)) return false;
  return (p->nsm + p->g.ntiles - 1) / p->g.ntiles + 1 <= p->adj_ch_cap;
}
int ct_pmax(const nf_plan* p) { return (p->g.ntiles + p->nsm - 1) / p->nsm + 2; }
// forward: the pieces whose iterate values (2 * TILE Reals each) fit behind the layout, and the layout with them
int ct_stage_pieces(const nf_plan* p) {
  const size_t lay = p->dtype == NF_C64 ? CtLayout<float>(p->g.A).bytes : CtLayout<double>(p->g.A).bytes;
  const size_t per = 2 * (size_t)TILE * real_size(p), room = 232448 - 4096 > lay ? 232448 - 4096 - lay : 0;
  return (int)std::min<size_t>(ct_pmax(p), room / per);
}
size_t ct_fwd_smem(const nf_plan* p) {
  const size_t lay = p->dtype == NF_C64 ? CtLayout<float>(p->g.A).bytes : CtLayout<double>(p->g.A).bytes;
  return lay + (size_t)ct_stage_pieces(p) * 2 * TILE * real_size(p);
}
int ct_part_buffer(nf_plan* p) {
  const size_t need = (size_t)p->nsm * ct_pmax(p) * TILE * 2 * real_size(p);
  if (need <= p->ctpart_bytes) return NF_OK;
  cudaFree(p->d_ctpart);
  p->d_ctpart = nullptr;
  p->ctpart_bytes = 0;
  if (int rc = dalloc(p, (char**)&p->d_ctpart, need)) return rc;
  p->ctpart_bytes = need;
  return NF_OK;
}
// rx-major batch order (KeyMap::rxmajor) when both phases of the batch run the CTA-tile kernels on one window
bool ct_rxmajor(const nf_plan* p, int B) {
  return p->ct_rx && B <= p->fwd_chunk && use_ct(p, B) && use_ct_adj(p, B);
}
// CtArgs of a window of `span` channels on G CTAs. kind 0: per-launch forward, 1: adjoint, 2: the persistent loop's
// forward (its last CTA sorts the next batch first and gets `loop_sort_disc` % less). The cuts equalise
// pairs + cost * pieces (cost in pairs; p->ct_cost_fwd / ct_cost_adj, 0: equal ranges) by bisection on the budget of a
// greedy walk; cached per kind (a plan's batches mostly repeat one span).
CtArgs ct_args(const nf_plan* p, int span, int kind, int G) {
  nf_plan::CtCache& cc = p->ct_cache[kind];
  const double cost = kind == 1 ? p->ct_cost_adj : p->ct_cost_fwd, disc = kind == 2 ? p->loop_sort_disc / 100.0 : 0.0;
  if (cc.span == span && cc.G == G && cc.cost == cost && cc.disc == disc) return cc.args;
  CtArgs c;
  c.W = (long long)p->g.ntiles * span;
  c.span = span;
  c.G = G;
  c.ns = kind == 1 ? 0 : ct_stage_pieces(p);
  for (int i = 0; i <= CT_GMAX; ++i) c.bnd[i] = (int)std::min<long long>(c.W, (long long)std::min(i, G) * c.W / G);
  const int pmax = ct_pmax(p), shmax = p->adj_ch_cap;
  std::vector<long long> bnd(G + 1, 0);
  // greedy walk with budget C per CTA: every piece costs `cost`, a piece is started only with room for `minp` pairs
  const double minp = CT_WARPS;
  auto walk = [&](double C) {
    long long u = 0;
    for (int i = 0; i < G; ++i) {
      bnd[i] = u;
      double budget = i == G - 1 ? C * (1.0 - disc) : C;
      while (u < c.W && budget >= cost + minp) {
        const long long rem = span - u % span;
        const long long take = std::min<long long>(rem, (long long)(budget - cost));
        u += take;
        budget -= cost + (double)take;
        if (take < rem) break;
      }
    }
    bnd[G] = u;
    return u >= c.W;
  };
  bool ok = G > 1 && (cost > 0 || disc > 0) && c.W / G > 4 * (long long)(cost + minp);
  if (ok) {
    double lo = (double)c.W / G, hi = 2.0 * ((double)c.W / G + cost * (pmax + 1)) / (1.0 - disc);
    ok = walk(hi);
    for (int it = 0; ok && it < 50 && hi - lo > 0.5; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (walk(mid)) hi = mid; else lo = mid;
    }
    if (ok) {
      walk(hi);
      bnd[G] = c.W;
      std::vector<int> share(p->g.ntiles, 0);
      for (int i = 0; ok && i < G; ++i) {  // within the parked-sum slots and the chunk-partial buffer
        const long long a = bnd[i], b = bnd[i + 1];
        if (b <= a) continue;  // the last CTAs may be left without pairs
        const int t0 = (int)(a / span), t1 = (int)((b - 1) / span);
        if (t1 - t0 + 1 > pmax) ok = false;
        for (int t = t0; t <= t1; ++t)
          if (++share[t] > shmax) ok = false;
      }
    }
    if (ok)
      for (int i = 1; i <= G; ++i) c.bnd[i] = (int)bnd[i];
  }
  cc.span = span;
  cc.G = G;
  cc.cost = cost;
  cc.disc = disc;
  cc.args = c;
  return c;
}

// Forward launch arguments of one window [w0, w1) of the staged flat batch (launch_forward, spgm_loop)
template <typename Real>
FwdArgs<Real> fwd_args(const nf_plan* p, const void* s, int w0, int w1, bool loop = false) {
  const int span = w1 - w0;
  FwdArgs<Real> a;
  a.g = p->g;
  a.tab = (const Real*)p->d_tab;
  a.D0 = p->d_D0;
  a.crec = p->d_crec;
  a.s = (const Real*)s;
  a.w0 = w0;
  a.w1 = w1;
  a.Q = channel_splits(p, span);
  a.part = (Real*)p->d_part;
  a.order = unit_order(p, (long long)p->g.ntiles * a.Q);
  tail_split(p, a.order, a.Q, std::max(1, span / p->min_chunk), a.t1, a.Q2);
  if ((loop ? p->loop_wave_fit : p->wave_fit) & 1) wave_fit(p, a.order, span, a.Q, a.t1, a.Q2);
  a.taper = (float)p->fwd_taper;
  return a;
}

// Adjoint (+ prox) arguments of the staged flat batch (launch_adjoint, spgm_loop)
template <typename Real>
AdjArgs<Real> adj_args(const nf_plan* p, void* gout, double scale, const void* s_in, void* s_out, double eta_over_b,
                       double alpha, bool loop = false) {
  AdjArgs<Real> a;
  a.g = p->g;
  a.tab = (const Real*)p->d_tab;
  a.D0 = p->d_D0;
  a.crec = p->d_crec;
  a.wrec = (const R2<Real>*)p->d_wrec;
  a.B = p->B;
  a.CH = adjoint_chunks(p);
  a.order = p->structured ? 0 : unit_order(p, (long long)p->g.ntiles * a.CH);
  a.t1 = p->g.ntiles;
  a.CH2 = a.CH;
  a.taper = (float)p->taper;
  if (!p->structured) {
    tail_split(p, a.order, a.CH, std::min<long long>(std::max(1, p->B / p->adj_min_chunk), p->adj_ch_cap), a.t1, a.CH2);
    if ((loop ? p->loop_wave_fit : p->wave_fit) & 2) wave_fit(p, a.order, std::min(p->B, p->adj_ch_cap), a.CH, a.t1, a.CH2);
  }
  a.gpart = (Real*)p->d_gpart;
  a.cnt = p->d_tilecnt;
  a.gout = (Real*)gout;
  a.scale = scale;
  a.s_in = (const Real*)s_in;
  a.s_out = (Real*)s_out;
  a.eta_over_b = eta_over_b;
  a.alpha = alpha;
  a.stat_part = p->d_stat_part;
  return a;
}

template <typename Real>
int launch_forward(nf_plan* p, const void* s, void* y, cudaStream_t st) {
  const size_t sm = fwd_smem(p);
  auto kern = p->exact ? fwd_kernel<Real, true> : fwd_kernel<Real, false>;
  CUDA_TRY(ensure_smem((const void*)kern, sm, true));
  for (int w0 = 0; w0 < p->B; w0 += p->fwd_chunk) {
    const int w1 = std::min(p->B, w0 + p->fwd_chunk);
    const int span = w1 - w0;
    const FwdArgs<Real> a = fwd_args<Real>(p, s, w0, w1);
    if (use_ct(p, span)) {  // part[tile][j] is the same either way (bit-identical per-(tile, channel) values)
      auto kct = p->exact ? fwd_ct_kernel<Real, true> : fwd_ct_kernel<Real, false>;
      const size_t smc = ct_fwd_smem(p);
      CUDA_TRY(ensure_smem((const void*)kct, smc));
      CUDA_TRY(launch_k(p->use_pdl, kct, dim3(p->nsm), dim3(CT_WARPS * 32), smc, st, a, ct_args(p, span, 0, p->nsm)));
    } else {
      const long long units = (long long)a.t1 * a.Q + (long long)(p->g.ntiles - a.t1) * a.Q2;
      CUDA_TRY(launch_k(p->use_pdl, kern, dim3((unsigned)((units + FWD_WARPS - 1) / FWD_WARPS)),
                        dim3(FWD_WARPS * 32), sm, st, a));
    }
    // two-level reduce: ~sqrt(rows) segments so both levels have short serial sums. The segment count
    // depends on the plan only, never on the span, so a channel's summation tree is the same in every
    // batch: forward_apply(s, subset=sub) == forward_apply(s)[sub] bit for bit (forward.py:17-18).
    const int nseg = p->fwd_nseg;
    CUDA_TRY(launch_k(p->use_pdl, fwd_reduce1_kernel<Real>, dim3((span + 255) / 256, nseg), dim3(256), 0, st,
                      (const Real*)p->d_part, p->fwd_gridx, span, nseg, p->d_tmp));
    if (int rc = launch_reduce2<Real>(p, span, nseg, w0, y, st, p->use_pdl, true)) return rc;
    p->launches += 3;
  }
  return NF_OK;
}

StructArgs struct_args(const nf_plan* p) {
  StructArgs sa;
  sa.fs = p->d_struct;
  sa.ts = p->d_struct + p->g.F;
  sa.rs = p->d_struct + p->g.F + p->g.T;
  sa.nf = p->snf;
  sa.nt = p->snt;
  sa.nr = p->snr;
  return sa;
}

template <typename Real, bool FWD>
size_t struct_smem(const nf_plan* p) {
  return SLayout<Real, FWD>::bytes(p->g.A);
}

// (f, t) row chunks per tile: enough blocks for the target, at least SW·4 rows each
int struct_splits(long long target_blocks, int ntiles, int rows) {
  long long q = (target_blocks + ntiles - 1) / ntiles;
  q = std::min<long long>(q, std::max(1, rows / (SW * 4)));
  return (int)std::max(1LL, q);
}

// tensor-core structured forward (c64): windows of whole frequencies, 2·tiles partial rows
int launch_forward_tc(nf_plan* p, const void* s, void* y, cudaStream_t st) {
  const StructArgs sa = struct_args(p);
  const int npr = (sa.nr + 15) / 16 * 16;
  const long long rows = 2LL * p->g.ntiles, per_f = (long long)sa.nt * sa.nr;
  // partial buffer: up to 2 GB, at least one frequency; windows of whole frequencies
  long long fwin = std::max(1LL, std::min<long long>(sa.nf, (2LL << 30) / (rows * 8 * per_f)));
  const int nseg = reduce_segments((int)rows);
  const long long nwins = (sa.nf + fwin - 1) / fwin;
  fwin = (sa.nf + nwins - 1) / nwins;  // balanced windows (16 = 8 + 8, not 14 + 2)
  const size_t need = (size_t)(rows * per_f * fwin);
  if ((size_t)nseg * per_f * fwin > p->tmp_elems) {  // one frequency's level-1 sums exceed the reduce buffer
    cudaFree(p->d_tmp);
    p->d_tmp = nullptr;
    p->tmp_elems = 0;
    int rc = dalloc(p, &p->d_tmp, (size_t)nseg * per_f * fwin * sizeof(double2));
    if (rc) return rc;
    p->tmp_elems = (size_t)nseg * per_f * fwin;
  }
  if (need > p->tcpart_elems) {
    cudaFree(p->d_tcpart);
    p->d_tcpart = nullptr;
    p->tcpart_elems = 0;
    int rc = dalloc(p, &p->d_tcpart, need * sizeof(float2));
    if (rc) return rc;
    p->tcpart_elems = need;
  }
  const bool stream = TcfLayout(npr, sa.nt + sa.nr, false).bytes > TC_SMEM_MAX;  // table too big to stage whole
  const uint32_t smem = TcfLayout(npr, sa.nt + sa.nr, stream).bytes;
  auto kern = stream ? (p->exact ? fwd_tc_kernel<true, true> : fwd_tc_kernel<false, true>)
                     : (p->exact ? fwd_tc_kernel<true, false> : fwd_tc_kernel<false, false>);
  CUDA_TRY(ensure_smem((const void*)kern, smem));
  for (int fa = 0; fa < sa.nf; fa += (int)fwin) {
    const int fb = std::min(sa.nf, fa + (int)fwin);
    FwdArgs<float> a;
    a.g = p->g;
    a.tab = (const float*)p->d_tab;
    a.D0 = p->d_D0;
    a.crec = nullptr;
    a.s = (const float*)s;
    a.w0 = (int)(fa * per_f);
    a.w1 = (int)(fb * per_f);
    a.Q = 1;
    a.order = 0;
    a.t1 = p->g.ntiles;
    a.Q2 = 1;
    a.taper = 0;
    a.part = nullptr;
    const int span = a.w1 - a.w0;
    // one CTA per SM, two per tile: split the window's frequencies for at least two waves
    const int fch = (int)std::min<long long>(fb - fa, std::max<long long>(1, (2LL * 148 + rows - 1) / rows));
    kern<<<(unsigned)(rows * fch), TC_THREADS, smem, st>>>(a, sa, p->d_kd, npr, fa, fb, fch, p->d_tcpart);
    CUDA_TRY(cudaGetLastError());
    fwd_reduce1_kernel<float><<<dim3((span + 255) / 256, nseg), 256, 0, st>>>((const float*)p->d_tcpart, (int)rows,
                                                                              span, nseg, p->d_tmp);
    CUDA_TRY(cudaGetLastError());
    if (int rc = launch_reduce2<float>(p, span, nseg, a.w0, y, st, false)) return rc;
    p->launches += 3;
  }
  return NF_OK;
}

bool use_tc_struct(const nf_plan* p, bool forward) {
  if (!p->structured || !p->use_tc || 2 * p->snt > TC_NMAX || p->snr > TC_RX_MAX) return false;
  const int amin = std::min(p->snt, p->snr);
  // the tensor core pays off once the contraction dominates the phasor work: both antenna
  // counts >= 24 and enough frequencies per tile (tools/time_structured.py crossover)
  if (!p->tc_force && !(amin >= 24 && p->snf * amin >= 192)) return false;
  if (forward) {  // the tcgen05 forward wins only on large batches: >= 40 antennas a side and
                  // >= 12 frequencies (full set: -10% vs FFMA); NFGPU_TC_FWD=1 takes it for every eligible batch
    if (!p->tc_force && !p->tc_fwd && !(amin >= 40 && p->snf >= 12)) return false;
    return p->snr <= 256 && TcfLayout((p->snr + 15) / 16 * 16, p->snt + p->snr, true).bytes <= TC_SMEM_MAX;
  }
  return TcLayout((2 * p->snt + 15) / 16 * 16, p->snt + p->snr, 2).bytes <= TC_SMEM_MAX;
}

template <typename Real>
int launch_forward_struct(nf_plan* p, const void* s, void* y, cudaStream_t st) {
  const size_t sm = struct_smem<Real, true>(p);
  auto kern = p->exact ? fwd_struct_kernel<Real, true> : fwd_struct_kernel<Real, false>;
  CUDA_TRY(ensure_smem((const void*)kern, sm, true));
  const StructArgs sa = struct_args(p);
  const int rows = sa.nf * sa.nt;
  const int win = std::max(1, p->fwd_chunk / sa.nr);  // rows per launch window (part buffer bound)
  for (int ua = 0; ua < rows; ua += win) {
    const int ub = std::min(rows, ua + win);
    FwdArgs<Real> a;
    a.g = p->g;
    a.tab = (const Real*)p->d_tab;
    a.D0 = p->d_D0;
    a.crec = nullptr;
    a.s = (const Real*)s;
    a.w0 = ua * sa.nr;
    a.w1 = ub * sa.nr;
    const int span = a.w1 - a.w0;
    a.Q = struct_splits(p->struct_target, p->g.ntiles, ub - ua);
    a.order = 0;
    a.t1 = p->g.ntiles;
    a.Q2 = a.Q;
    a.taper = 0;
    a.part = (Real*)p->d_part;
    kern<<<(unsigned)((long long)p->g.ntiles * a.Q), SW * 32, sm, st>>>(a, sa, p->d_kd);
    CUDA_TRY(cudaGetLastError());
    const int nseg = p->fwd_nseg;
    fwd_reduce1_kernel<Real><<<dim3((span + 255) / 256, nseg), 256, 0, st>>>((const Real*)p->d_part, p->fwd_gridx,
                                                                             span, nseg, p->d_tmp);
    CUDA_TRY(cudaGetLastError());
    if (int rc = launch_reduce2<Real>(p, span, nseg, a.w0, y, st, false)) return rc;
    p->launches += 3;
  }
  return NF_OK;
}

template <typename Real, bool PROX>
int launch_adjoint(nf_plan* p, const void* r, const void* ymeas, void* gout, double scale, const void* s_in,
                   void* s_out, double eta_over_b, double alpha, double* stats, cudaStream_t st) {
  const int nblk = (p->B + 255) / 256;
  CUDA_TRY(launch_k(p->use_pdl, resid_kernel<Real>, dim3(nblk), dim3(256), 0, st, p->d_sm, p->d_spos, p->d_sf, p->B,
                    (const Real*)r, (const Real*)ymeas, p->d_pulse, (R2<Real>*)p->d_wrec, p->d_dpart));
  AdjArgs<Real> a = adj_args<Real>(p, gout, scale, s_in, s_out, eta_over_b, alpha);
  if constexpr (std::is_same<Real, float>::value) {
    const int npad = (2 * p->snt + 15) / 16 * 16;
    if (use_tc_struct(p, false)) {
      const StructArgs sa = struct_args(p);
      const int nch = (sa.nr + TC_RCH - 1) / TC_RCH;
      tc_bprep_kernel<<<sa.nf * nch, 256, 0, st>>>(sa, (const float2*)p->d_wrec, npad, nch, p->d_bimg);
      CUDA_TRY(cudaGetLastError());
      // one CTA per SM, two per tile (halves); split frequencies for at least two waves
      int fch = (int)std::min<long long>(sa.nf, std::max<long long>(1, (2LL * 148 + 2 * p->g.ntiles - 1) /
                                                                          (2 * p->g.ntiles)));
      fch = std::max(1, std::min(fch, p->adj_ch_cap / 2));
      a.CH = 2 * fch;
      int ns = TC_NS;  // as many pipeline stages as fit next to the table
      while (ns > 2 && TcLayout(npad, sa.nt + sa.nr, ns).bytes > TC_SMEM_MAX) --ns;
      const uint32_t smem = TcLayout(npad, sa.nt + sa.nr, ns).bytes;
      auto kern = p->exact ? adj_tc_kernel<PROX, true> : adj_tc_kernel<PROX, false>;
      CUDA_TRY(ensure_smem((const void*)kern, smem));
      kern<<<(unsigned)(p->g.ntiles * a.CH), TC_THREADS, smem, st>>>(a, sa, p->d_kd, p->d_bimg, npad, nch, fch, ns);
      CUDA_TRY(cudaGetLastError());
      p->launches += 3;
      if (PROX) {
        stats_reduce_kernel<<<1, 256, 0, st>>>(p->d_stat_part, p->g.ntiles, p->d_dpart, nblk, stats);
        CUDA_TRY(cudaGetLastError());
        p->launches += 1;
      }
      return NF_OK;
    }
  }
  if (p->structured) {
    const StructArgs sa = struct_args(p);
    a.CH = std::min(struct_splits(p->struct_target, p->g.ntiles, sa.nf * sa.nt), p->adj_ch_cap);
    const size_t sm = struct_smem<Real, false>(p);
    auto kern = p->exact ? adj_struct_kernel<Real, PROX, true> : adj_struct_kernel<Real, PROX, false>;
    CUDA_TRY(ensure_smem((const void*)kern, sm, true));
    kern<<<(unsigned)(p->g.ntiles * a.CH), SW * 32, sm, st>>>(a, sa, p->d_kd);
  } else if (use_ct_adj(p, p->B)) {
    if (int rc = ct_part_buffer(p)) return rc;
    auto kct = p->exact ? adj_ct_kernel<Real, PROX, true> : adj_ct_kernel<Real, PROX, false>;
    const size_t smc = CtLayout<Real>(p->g.A).bytes;
    CUDA_TRY(ensure_smem((const void*)kct, smc));
    CUDA_TRY(launch_k(p->use_pdl, kct, dim3(p->nsm), dim3(CT_WARPS * 32), smc, st, a, ct_args(p, p->B, 1, p->nsm),
                      (Real*)p->d_ctpart, ct_pmax(p)));
  } else {
    const size_t sm = adj_smem(p);
    auto kern = p->exact ? adj_kernel<Real, PROX, true> : adj_kernel<Real, PROX, false>;
    CUDA_TRY(ensure_smem((const void*)kern, sm, true));
    const int units = a.t1 * a.CH + (p->g.ntiles - a.t1) * a.CH2;
    CUDA_TRY(launch_k(p->use_pdl, kern, dim3((units + ADJ_WARPS - 1) / ADJ_WARPS), dim3(ADJ_WARPS * 32), sm, st, a));
  }
  CUDA_TRY(cudaGetLastError());
  p->launches += 2;
  if (PROX) {
    CUDA_TRY(launch_k(p->use_pdl, stats_reduce_kernel, dim3(1), dim3(256), 0, st, (const double*)p->d_stat_part,
                      p->g.ntiles, (const double*)p->d_dpart, nblk, stats));
    p->launches += 1;
  }
  return NF_OK;
}

// NFGPU_LOOP_PROFILE: phase time stamps of CTA 0 into a plan buffer (nf_loop_profile reads them back)
int loop_profile_buffer(nf_plan* p, int K, LoopArgs& la) {
  la.prof = nullptr;
  la.prof_cta = 0;
  const char* env = std::getenv("NFGPU_LOOP_PROFILE");
  if (!env) return NF_OK;
  la.prof_cta = std::atoi(env) == 2;
  const size_t need = (size_t)K * (LOOP_PROF + (la.prof_cta ? 2 * LOOP_PROF_CTA : 0)) + (la.prof_cta ? LOOP_PROF_CTA : 0);
  if (need > p->loop_prof_elems) {
    cudaFree(p->d_loop_prof);
    p->d_loop_prof = nullptr;
    p->loop_prof_elems = 0;
    if (int rc = dalloc(p, &p->d_loop_prof, need * sizeof(unsigned long long))) return rc;
    p->loop_prof_elems = need;
  }
  la.prof = p->d_loop_prof;
  return NF_OK;
}

template <typename Real>
int launch_tiny_loop(nf_plan* p, const int32_t* table, int K, uint64_t seed, uint64_t iter0, int B, const void* ymeas,
                     void* s_a, void* s_b, double eta_over_b, double alpha, double tol, long long budget_ns,
                     double* rec, int* state, cudaStream_t st) {
  int dev = 0, nsm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const Geo& g = p->g;
  const int nvb = (int)((p->nvox + 255) / 256);
  int jc = (int)std::max(1LL, std::min<long long>(TINY_JC, ((long long)B * nvb + nsm - 1) / nsm));
  int cc = std::max(1, std::min(B, nsm / std::max(1, nvb)));
  if (const char* e = std::getenv("NFGPU_TINY_JC")) jc = std::max(1, std::min(TINY_JC, std::atoi(e)));
  if (const char* e = std::getenv("NFGPU_TINY_CC")) cc = std::max(1, std::min(B, std::atoi(e)));
  const size_t b_part = sizeof(double2) * (size_t)nvb * B, b_w = sizeof(double) * (size_t)B, b_ch = 0,
               b_g = sizeof(double2) * (size_t)cc * nvb * 256,
               b_cnt = sizeof(int) * (size_t)nvb, b_st = sizeof(double) * 4 * (size_t)nvb;
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t need = al(b_part) + al(b_w) + al(b_ch) + al(b_g) + al(b_cnt) + al(b_st);
  if (need > p->tiny_bytes) {
    cudaFree(p->d_tiny);
    p->d_tiny = nullptr;
    p->tiny_bytes = 0;
    if (int rc = dalloc(p, (char**)&p->d_tiny, need)) return rc;
    CUDA_TRY(cudaMemset(p->d_tiny, 0, need));
    p->tiny_bytes = need;
  }
  char* base = (char*)p->d_tiny;
  TinyArgs ta;
  ta.ant = p->d_ant;
  ta.kd = p->d_kd;
  for (int i = 0; i < 3; ++i) {
    ta.corner[i] = g.corner[i];
    ta.sp[i] = g.sp[i];
  }
  ta.nx = g.nx;
  ta.ny = g.ny;
  ta.nzs = g.nzs;
  ta.zb = g.zb;
  ta.T = g.T;
  ta.R = g.R;
  ta.nvb = nvb;
  ta.jc = jc;
  ta.cc = cc;
  ta.chunk_max = (B + cc - 1) / cc;
  // the per-voxel-block arrays first (their offsets depend on the plan only), then the batch-sized ones
  ta.vbcnt = (int*)base;  // zero between iterations (reset by the last arriver; cleared per launch below)
  base += al(b_cnt);
  ta.stat_part = (double*)base;
  base += al(b_st);
  ta.part = (double2*)base;
  base += al(b_part);
  ta.e2 = (double*)base;
  base += al(b_w);
  base += al(b_ch);
  ta.gpart = (double2*)base;
  if (!p->d_loopbar) {
    int rc = dalloc(p, &p->d_loopbar, 4 * sizeof(unsigned));
    if (rc) return rc;
    CUDA_TRY(cudaMemset(p->d_loopbar, 0, 4 * sizeof(unsigned)));
  }
  LoopArgs la = {};
  la.km = p->km;
  la.M = p->M;
  la.B = B;
  la.K = K;
  int bits = 2;
  while ((1LL << bits) < p->M) bits += 2;
  la.hb = bits / 2;
  la.idx_table = table;
  la.seed = seed;
  la.iter0 = iter0;
  la.kd = p->d_kd;
  la.pulse = p->d_pulse;
  la.ymeas = ymeas;
  la.dpart = p->d_dpart;
  la.tol = tol;
  la.budget_ns = budget_ns;
  la.eta_over_b = eta_over_b;
  la.alpha = alpha;
  la.rec = rec;
  la.state = state;
  la.bar = p->d_loopbar;
  la.s_a = s_a;
  la.s_b = s_b;
  la.prev_state = p->loop_prev;
  la.fold = p->loop_fold;
  if (int rc = loop_profile_buffer(p, K, la)) return rc;
  const size_t smem = (size_t)ta.chunk_max * (sizeof(double2) + sizeof(int4));
  auto kern = tiny_loop_kernel<Real>;
  CUDA_TRY(ensure_smem((const void*)kern, smem));
  CUDA_TRY(cudaMemsetAsync(state, 0, 3 * sizeof(int), st));
  CUDA_TRY(cudaMemsetAsync(p->d_loopbar, 0, sizeof(unsigned), st));  // the grid barrier's arrival counter
  CUDA_TRY(cudaMemsetAsync(ta.vbcnt, 0, b_cnt, st));
  if (std::getenv("NFGPU_VERBOSE"))
    std::fprintf(stderr, "nf_spgm_loop: tiny_loop_kernel, %d CTAs x 256 threads, B=%d, K=%d\n", nsm, B, K);
  void* args[] = {&la, &ta};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(nsm), dim3(256), args, smem, st));
  p->B = B;
  p->structured = false;
  p->launches += 1;
  return NF_OK;
}

template <typename Real>
int launch_spgm_loop(nf_plan* p, const int32_t* table, int K, uint64_t seed, uint64_t iter0, int B, const void* ymeas,
                     void* s_a, void* s_b, double eta_over_b, double alpha, double tol, long long budget_ns,
                     double* rec, int* state, cudaStream_t st) {
  const char* tiny_env = std::getenv("NFGPU_TINY");  // read per launch: "0" keeps small problems here
  if ((!tiny_env || std::atoi(tiny_env) != 0) && (long long)B * p->nvox <= TINY_MAX_ENTRIES)
    return launch_tiny_loop<Real>(p, table, K, seed, iter0, B, ymeas, s_a, s_b, eta_over_b, alpha, tol, budget_ns,
                                  rec, state, st);
  // the forward phase on the CTA-tile kernel (as nf_forward would run it; its values are bit-identical either way)
  // when its layout fits next to 16 warp regions. The loop's batches are flat: the plan's structured flag (left by
  // an earlier staged batch) must not steer the choice away from what nf_adjoint_prox runs on a flat batch.
  p->structured = false;
  bool ct = use_ct(p, B);
  const bool cta = ct && use_ct_adj(p, B);
  auto pick = [&](bool f, bool a) {
    if (p->exact)
      return a ? spgm_loop_kernel<Real, true, 3> : f ? spgm_loop_kernel<Real, true, 1> : spgm_loop_kernel<Real, true, 0>;
    return a ? spgm_loop_kernel<Real, false, 3> : f ? spgm_loop_kernel<Real, false, 1> : spgm_loop_kernel<Real, false, 0>;
  };
  auto kern = pick(ct, cta);
  size_t wb = std::max(fwd_warp_bytes<Real>(p->g.Tg, p->g.A), warp_smem_bytes<Real>(p->g.Tg, p->g.A));
  wb = (wb + 15) & ~(size_t)15;
  cudaFuncAttributes fattr;
  CUDA_TRY(cudaFuncGetAttributes(&fattr, kern));
  const size_t SMEM_DYN_MAX = 232448 - fattr.sharedSizeBytes;  // 227 KB per block (opt-in) beside the static part
  int nw = 16;  // warps per CTA: 16, 12 or 8 (multiples of 4 keep the 256-thread groups of P3 / P5)
  if (!cta) {  // the warp-unit adjoint's regions (the CTA-tile kernels of both phases use CtLayout only)
    while (nw > 8 && (size_t)nw * wb > SMEM_DYN_MAX) nw -= 4;
    if ((size_t)nw * wb > SMEM_DYN_MAX)
      return fail(NF_ERR_STATE, "persistent loop: shared memory layout does not fit");
  }
  // P0 rank sort: keys + order (LOOP_SORT_MAX ints each), then the key bitmap and its word prefix counts
  const size_t kwords = ((size_t)p->KS + 31) / 32;
  const bool bitmap = (size_t)LOOP_SORT_MAX * 8 + kwords * 8 <= SMEM_DYN_MAX;
  const size_t sort_bytes = (size_t)LOOP_SORT_MAX * 8 + (bitmap ? kwords * 8 : 0);
  size_t smem = std::max(sort_bytes, (size_t)(4 * 256 + 16) * sizeof(double));
  if (!cta) smem = std::max(smem, (size_t)nw * wb);
  if (ct && !cta && nw != 16) {  // CTA-tile forward beside the warp-unit adjoint needs 16 warps (its values are the same)
    ct = false;
    kern = pick(false, false);
  }
  const bool ct_adjoint_on = cta;
  if (ct) smem = std::max(smem, ct_fwd_smem(p));
  int stage_tiles = 0;
  {  // the reduce phase's segment sums [nseg][channels per CTA], and behind them the staging buffer for the CTA's
    // partials [tiles per chunk][channels per CTA]: within the layout the other phases need anyway (or 64 KB)
    const int nred = std::max(1, p->nsm - 1);
    const size_t jc = (size_t)(B + nred - 1) / nred;
    const size_t seg_bytes = (size_t)p->fwd_nseg * jc * sizeof(double2);
    smem = std::max(smem, seg_bytes);
    const size_t budget = std::min(std::max(smem, (size_t)65536), SMEM_DYN_MAX), per_tile = jc * 2 * sizeof(Real);
    if (budget > seg_bytes) stage_tiles = (int)std::min<size_t>(p->g.ntiles, (budget - seg_bytes) / per_tile);
    if (stage_tiles < 16 && stage_tiles < p->g.ntiles) stage_tiles = 0;
    if (stage_tiles > 0) smem = std::max(smem, seg_bytes + (size_t)stage_tiles * per_tile);
  }
  if (smem > SMEM_DYN_MAX) return fail(NF_ERR_STATE, "persistent loop: shared memory layout does not fit");
  if (ct_adjoint_on)
    if (int rc = ct_part_buffer(p)) return rc;
  CUDA_TRY(ensure_smem((const void*)kern, smem));
  int dev = 0, nsm = 0, per_sm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem));
  if (per_sm < 1) return fail(NF_ERR_STATE, "persistent loop: one CTA per SM does not fit");
  if (!p->d_loopbar) {  // {barrier arrivals, barrier generation, forward unit counter, adjoint unit counter}
    int rc = dalloc(p, &p->d_loopbar, 4 * sizeof(unsigned));
    if (rc) return rc;
    CUDA_TRY(cudaMemset(p->d_loopbar, 0, 4 * sizeof(unsigned)));
  }
  p->B = B;
  p->structured = false;
  LoopArgs la;
  la.km = cta && ct_rxmajor(p, B) ? p->km_rx : p->km;  // the order nf_batch_prepare gives this batch
  la.M = p->M;
  la.B = B;
  la.K = K;
  la.nseg = p->fwd_nseg;
  int bits = 2;
  while ((1LL << bits) < p->M) bits += 2;
  la.hb = bits / 2;
  la.idx_table = table;
  la.seed = seed;
  la.iter0 = iter0;
  la.kd = p->d_kd;
  la.pulse = p->d_pulse;
  la.ymeas = ymeas;
  la.ymeas_f64 = std::is_same<Real, double>::value ? 1 : 0;
  {  // sorted channel records [2 parities][B]
    const size_t n = (size_t)2 * B;
    const size_t need = n * (sizeof(ChanRec) + 3 * sizeof(int) + 2 * sizeof(double2)) + 16;
    if (need > p->loop_priv_bytes) {
      cudaFree(p->d_loop_priv);
      p->d_loop_priv = nullptr;
      p->loop_priv_bytes = 0;
      if (int rc = dalloc(p, (char**)&p->d_loop_priv, need)) return rc;
      p->loop_priv_bytes = need;
    }
    char* b = (char*)p->d_loop_priv;
    la.yrec = (double2*)b;
    b += n * 2 * sizeof(double2);
    la.crec = (ChanRec*)b;
    b += n * sizeof(ChanRec);
    la.sm = (int*)b;
    b += n * sizeof(int);
    la.spos = (int*)b;
    b += n * sizeof(int);
    la.sf = (int*)b;
  }
  la.tmp = p->d_tmp;
  la.dpart = p->d_dpart;
  la.stat_part = p->d_stat_part;
  la.tol = tol;
  la.budget_ns = budget_ns;
  la.rec = rec;
  la.state = state;
  la.bar = p->d_loopbar;
  la.ctr = (int*)p->d_loopbar + 2;
  la.s_a = s_a;
  la.s_b = s_b;
  la.prev_state = p->loop_prev;
  la.fold = p->loop_fold;
  la.warp_bytes = wb;
  la.kwords = bitmap ? (int)kwords : 0;
  la.stage_tiles = stage_tiles;
  if (int rc = loop_profile_buffer(p, K, la)) return rc;
  FwdArgs<Real> fa = fwd_args<Real>(p, s_a, 0, B, true);
  AdjArgs<Real> aa = adj_args<Real>(p, nullptr, 0, s_a, s_b, eta_over_b, alpha, true);
  CUDA_TRY(cudaMemsetAsync(state, 0, 3 * sizeof(int), st));
  CUDA_TRY(cudaMemsetAsync(p->d_loopbar, 0, sizeof(unsigned), st));  // the grid barrier's arrival counter
  CtArgs ca = ct_args(p, B, 1, nsm);
  la.ctpart = p->d_ctpart;
  la.ctpmax = ct_pmax(p);
  if (std::getenv("NFGPU_VERBOSE"))
    std::fprintf(stderr, "nf_spgm_loop: spgm_loop_kernel (%s forward, %s adjoint), %d CTAs x %d warps, %zu B shared, "
                 "B=%d, K=%d, ctpart %p (%zu B, pmax %d)\n", ct ? "CTA-tile" : "warp-unit",
                 ct_adjoint_on ? "CTA-tile" : "warp-unit", nsm, nw, smem, B, K, p->d_ctpart, p->ctpart_bytes,
                 ct_pmax(p));
  CtArgs cf = ct_args(p, B, 2, nsm);  // forward ranges: the sorting CTA (the last) gets loop_sort_disc % less
  void* args[] = {&la, &fa, &aa, &ca, &cf};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(nsm), dim3(nw * 32), args, smem, st));
  p->loop_threads = nw * 32;
  p->launches += 1;
  return NF_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* nf_last_error(void) { return g_err.c_str(); }

int nf_plan_create(const double* tx_xyz, int n_tx, const double* rx_xyz, int n_rx, const double* freq_hz,
                   const double* pulse_reim, int n_f, double c, const double corner[3], const double spacing[3],
                   const int dims[3], int z_begin, int z_end, int dtype, int max_batch, nf_plan** out) {
  if (!out) return fail(NF_ERR_ARG, "out is null");
  *out = nullptr;
  if (!tx_xyz || !rx_xyz || !freq_hz || !pulse_reim || !corner || !spacing || !dims)
    return fail(NF_ERR_ARG, "null geometry pointer");
  if (n_tx < 1 || n_rx < 1 || n_f < 1) return fail(NF_ERR_ARG, "n_tx, n_rx, n_f must be >= 1");
  if (n_rx > R_MAX) return fail(NF_ERR_ARG, "at most 32767 receivers per plan");
  if (n_tx > TGROUPS_MAX * 2) return fail(NF_ERR_ARG, "at most 1022 transmitters per plan");
  if (!(c > 0) || !std::isfinite(c)) return fail(NF_ERR_ARG, "speed of light must be positive and finite");
  if (dtype != NF_C64 && dtype != NF_C128) return fail(NF_ERR_ARG, "dtype must be NF_C64 or NF_C128");
  for (int i = 0; i < 3; ++i)
    if (dims[i] < 1) return fail(NF_ERR_ARG, "dims must be >= 1");
  if (z_begin < 0 || z_end > dims[2] || z_begin >= z_end) return fail(NF_ERR_ARG, "bad z slab");
  const long long M = (long long)n_f * n_tx * n_rx;
  if (M > INT32_MAX / 8) return fail(NF_ERR_ARG, "too many channels");
  if (max_batch < 1 || max_batch > M) max_batch = (int)M;
  nf_plan* p = new nf_plan();
  p->dtype = dtype;
  p->M = (int)M;
  p->max_batch = max_batch;
  p->c = c;
  Geo& g = p->g;
  g.T = n_tx;
  g.R = n_rx;
  g.A = n_tx + n_rx;
  g.F = n_f;
  g.nx = dims[0];
  g.ny = dims[1];
  g.nzs = z_end - z_begin;
  g.zb = z_begin;
  g.ntx = (g.nx + TILE_X - 1) / TILE_X;
  g.nty = (g.ny + TILE_Y - 1) / TILE_Y;
  g.ntz = (g.nzs + TILE_Z - 1) / TILE_Z;
  g.ntiles = g.ntx * g.nty * g.ntz;
  // tx-group size: c128 rows are twice as wide, so 2-transmitter groups keep 12 warps per SM instead of 8
  // (Large c128 step 240 -> 280 Gentry/s, 1/8 slab 228 -> 259; Medium 189 -> 182; env NFGPU_TG_C128)
  int tg_max = TG_MAX;
  if (dtype == NF_C128) {
    tg_max = std::min(2, TG_MAX);
    if (const char* e = std::getenv("NFGPU_TG_C128")) tg_max = std::max(1, std::min(TG_MAX, std::atoi(e)));
  }
  g.ng = (n_tx + tg_max - 1) / tg_max;
  g.Tg = (n_tx + g.ng - 1) / g.ng;
  g.tg_mul = (65536 + g.Tg - 1) / g.Tg;
  if (g.ng > TGROUPS_MAX) {
    delete p;
    return fail(NF_ERR_ARG, "too many transmitter groups");
  }
  for (int i = 0; i < 3; ++i) {
    g.corner[i] = corner[i];
    g.sp[i] = spacing[i];
  }
  p->nvox = (int64_t)g.nx * g.ny * g.nzs;
  {  // every kernel keeps the tile's anchor distances of all T + R antennas in shared memory
    const size_t lim = 227 * 1024;
    const size_t need = std::max({fwd_smem(p), adj_smem(p),
                                  dtype == NF_C64 ? struct_smem<float, true>(p) : struct_smem<double, true>(p),
                                  dtype == NF_C64 ? struct_smem<float, false>(p) : struct_smem<double, false>(p)});
    if (need > lim) {
      delete p;
      return fail(NF_ERR_ARG, "too many antennas for the kernels' shared-memory layout (" + std::to_string(need) +
                                  " bytes per block)");
    }
  }
  p->km = KeyMap{g.T, g.R, g.F, g.Tg, g.ng, 0};
  p->km_rx = KeyMap{g.T, g.R, g.F, g.Tg, g.ng, 1};
  p->KS = g.ng * g.R * g.Tg * g.F;
  p->ksblocks = (p->KS + 1023) / 1024;
  p->fwd_gridx = g.ntiles;  // rows of the forward partial buffer (one per tile)
  p->fwd_nseg = reduce_segments(p->fwd_gridx);
  {
    // |x| = |base + (f/c)(δT + δR)| <= 1/2 + (f_max/c) * 2 * (tile half-diagonal), since |δ| <= distance
    // from the tile centre to the voxel (triangle inequality).
    const double hx = 0.5 * (TILE_X - 1) * spacing[0], hy = 0.5 * (TILE_Y - 1) * spacing[1];
    const double hz = 0.5 * (TILE_Z - 1) * spacing[2];
    double fmax = 0;
    for (int i = 0; i < n_f; ++i) fmax = std::max(fmax, std::fabs(freq_hz[i]));
    p->phase_bound_rev = 0.5 + fmax / c * 2.0 * std::sqrt(hx * hx + hy * hy + hz * hz);
    p->exact = dtype != NF_C64 || p->phase_bound_rev > EXACT_FREE_REV || std::getenv("NFGPU_FORCE_EXACT");
  }
  if (const char* e = std::getenv("NFGPU_STRUCT_TARGET")) p->struct_target = std::max(1LL, std::atoll(e));
  if (const char* e = std::getenv("NFGPU_MIN_CHUNK")) p->min_chunk = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("NFGPU_ADJ_MIN_CHUNK")) p->adj_min_chunk = std::max(1, std::atoi(e));
  const size_t rs = real_size(p);
  // Work-unit order (unit_coords / chunk_bound). Chunk-major with tapered chunks ends a launch on
  // short units (1/8 Large slab +2.2%, 1/4 slab +2.3%), but a tile's chunks are then far apart,
  // so its table rows are re-read from DRAM unless the table stays in L2 (full Large: 1.5 -> 5.3 GB
  // per forward for +0.9%). Tile-major equal chunks above NFGPU_L2_TABLE_MB; env NFGPU_CHUNK_ORDER.
  p->chunk_order = rs * (size_t)g.ntiles * g.A * TABW <= ((size_t)NFGPU_L2_TABLE_MB << 20) ? 1 : 0;
  if (const char* e = std::getenv("NFGPU_CHUNK_ORDER")) p->chunk_order = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("NFGPU_TAIL")) p->tail_split = std::atoi(e) != 0;
  if (const char* e = std::getenv("NFGPU_WAVE_FIT")) p->wave_fit = std::atoi(e);
  if (const char* e = std::getenv("NFGPU_LOOP_WAVE_FIT")) p->loop_wave_fit = std::atoi(e);
  if (const char* e = std::getenv("NFGPU_CT_COST_FWD")) p->ct_cost_fwd = std::max(0.0, std::atof(e));
  if (const char* e = std::getenv("NFGPU_CT_COST_ADJ")) p->ct_cost_adj = std::max(0.0, std::atof(e));
  if (const char* e = std::getenv("NFGPU_SORT_DISC")) p->loop_sort_disc = std::max(0.0, std::min(90.0, std::atof(e)));
  if (const char* e = std::getenv("NFGPU_FIT_MIN_WAVES")) p->fit_min_waves = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("NFGPU_TAIL_FACTOR")) p->tail_factor = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("NFGPU_TAIL_WAVES")) p->tail_waves = std::max(0.0, std::atof(e));
  if (const char* e = std::getenv("NFGPU_TAPER")) p->taper = std::min(0.49, std::max(0.0, std::atof(e)));
  if (const char* e = std::getenv("NFGPU_FWD_TAPER")) p->fwd_taper = std::min(0.49, std::max(0.0, std::atof(e)));
  // Warp units per launch. Chunk-major (L2-resident tables): forward four waves, adjoint ~3.2 waves (1/8 Large
  // slab 15 chunks 0.327 ms vs 10 chunks 0.351 ms, 1/4 slab 8 chunks 0.610 vs 5 chunks 0.644). Tile-major:
  // 12288 units (~5.2 waves) for both, i.e. 3 chunks per tile on full Large and 6 on the 1/2 slab (forward
  // 1.278 -> 1.262 ms, adjoint 1.148 -> 1.139 ms vs 5 chunks; the full problem is flat between 3 and 4).
  p->fwd_target = p->chunk_order ? 148LL * 16 * 4 : 12288;
  p->adj_target = p->chunk_order ? 148LL * 16 * 16 / 5 : 12288;
  if (const char* e = std::getenv("NFGPU_FWD_TARGET")) p->fwd_target = std::max(1LL, std::atoll(e));
  if (const char* e = std::getenv("NFGPU_ADJ_TARGET")) p->adj_target = std::max(1LL, std::atoll(e));
  {
    // bound the forward partial buffer to ~512 MB
    long long ch = (512LL << 20) / ((long long)p->fwd_gridx * 2 * rs);
    ch = std::max<long long>(ch, 1024) / 256 * 256;  // windows start at multiples of 256 channels (peer all-reduce)
    ch = std::min<long long>(ch, max_batch);
    p->fwd_chunk = (int)ch;
    // bound the adjoint chunk partials to ~256 MB
    const long long per = (long long)g.ntiles * TILE * 2 * rs;
    p->adj_ch_cap = (int)std::max<long long>(1, std::min<long long>(64, (256LL << 20) / per));
  }

  int rc;
  std::vector<double> ant(3 * (size_t)g.A);
  std::memcpy(ant.data(), tx_xyz, sizeof(double) * 3 * n_tx);
  std::memcpy(ant.data() + 3 * n_tx, rx_xyz, sizeof(double) * 3 * n_rx);
  std::vector<double> kd(n_f);
  std::vector<float> kf32(n_f);
  for (int i = 0; i < n_f; ++i) {
    kd[i] = freq_hz[i] / c;
    kf32[i] = (float)kd[i];
  }
  // level-1 sums of one forward window: fwd_nseg rows of fwd_chunk channels (the tensor-core forward grows
  // it for its frequency windows on first use)
  p->tmp_elems = (size_t)p->fwd_nseg * p->fwd_chunk;
  const size_t nred = p->tmp_elems;
#define ALLOC(ptr, bytes)                  \
  if ((rc = dalloc(p, &(ptr), (bytes)))) { \
    free_plan(p);                          \
    return rc;                             \
  }
  ALLOC(p->d_ant, sizeof(double) * 3 * g.A);
  ALLOC(p->d_kd, sizeof(double) * n_f);
  ALLOC(p->d_kf, rs * n_f);
  ALLOC(p->d_pulse, sizeof(double) * 2 * n_f);
  ALLOC(p->d_tab, rs * (size_t)g.ntiles * g.A * TABW);
  ALLOC(p->d_D0, sizeof(double) * (size_t)g.ntiles * g.A);
  ALLOC(p->d_pos_of_key, sizeof(int) * (size_t)p->KS);
  ALLOC(p->d_cnt, sizeof(int) * (size_t)p->ksblocks);
  ALLOC(p->d_sm, sizeof(int) * (size_t)max_batch);
  ALLOC(p->d_spos, sizeof(int) * (size_t)max_batch);
  ALLOC(p->d_crec, sizeof(ChanRec) * (size_t)max_batch);
  ALLOC(p->d_sf, sizeof(int) * (size_t)max_batch);
  ALLOC(p->d_wrec, 2 * rs * (size_t)max_batch);
  ALLOC(p->d_dpart, sizeof(double) * ((size_t)max_batch / 256 + 2));
  ALLOC(p->d_part, 2 * rs * (size_t)p->fwd_gridx * p->fwd_chunk);
  ALLOC(p->d_tmp, sizeof(double2) * nred);
  ALLOC(p->d_gpart, 2 * rs * (size_t)p->adj_ch_cap * g.ntiles * TILE);
  ALLOC(p->d_tilecnt, sizeof(int) * (size_t)g.ntiles);
  ALLOC(p->d_stat_part, sizeof(double) * 4 * (size_t)g.ntiles);
  ALLOC(p->d_iter, sizeof(unsigned long long));
  ALLOC(p->d_struct, sizeof(int) * (size_t)(n_f + n_tx + n_rx));
  p->use_tc = NFGPU_TC && dtype == NF_C64 && 2 * n_tx <= TC_NMAX;
  if (const char* e = std::getenv("NFGPU_TC")) {
    p->use_tc = p->use_tc && std::atoi(e) != 0;
    p->tc_force = std::atoi(e) == 2;
  }
  if (const char* e = std::getenv("NFGPU_TC_FWD")) p->tc_fwd = std::atoi(e) != 0;
  if (const char* e = std::getenv("NFGPU_PDL")) p->use_pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("NFGPU_CT")) p->ct_mode = std::atoi(e);
  if (const char* e = std::getenv("NFGPU_CT_MIN")) p->ct_min_pairs = std::max(1LL, std::atoll(e));
  if (const char* e = std::getenv("NFGPU_CT_ADJ")) p->ct_adj = std::atoi(e);
  if (const char* e = std::getenv("NFGPU_CT_RXMAJOR")) p->ct_rx = std::atoi(e);
  {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      p->nsm = nsm;
  }
  if (p->use_tc) {
    const size_t npad_max = (size_t)((2 * n_tx + 15) / 16) * 16;
    ALLOC(p->d_bimg, (size_t)n_f * ((n_rx + TC_RCH - 1) / TC_RCH) * npad_max * (2 * TC_RCH) * 4 * 2);
  }
#undef ALLOC
  auto cp = [&](void* dst, const void* src, size_t n) -> int {
    cudaError_t e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(NF_ERR_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
    return NF_OK;
  };
  if ((rc = cp(p->d_ant, ant.data(), sizeof(double) * 3 * g.A)) ||
      (rc = cp(p->d_kd, kd.data(), sizeof(double) * n_f)) ||
      (rc = cp(p->d_kf, dtype == NF_C64 ? (const void*)kf32.data() : (const void*)kd.data(), rs * n_f)) ||
      (rc = cp(p->d_pulse, pulse_reim, sizeof(double) * 2 * n_f))) {
    free_plan(p);
    return rc;
  }
  if (cudaMemset(p->d_pos_of_key, 0xff, sizeof(int) * (size_t)p->KS) != cudaSuccess ||
      cudaMemset(p->d_tilecnt, 0, sizeof(int) * (size_t)g.ntiles) != cudaSuccess ||
      cudaMemset(p->d_iter, 0, sizeof(unsigned long long)) != cudaSuccess) {
    free_plan(p);
    return fail(NF_ERR_CUDA, "cudaMemset");
  }
  dim3 grid(g.ntiles, g.A);
  if (dtype == NF_C64)
    build_table_kernel<float><<<grid, 32>>>(g, p->d_ant, (float*)p->d_tab, p->d_D0);
  else
    build_table_kernel<double><<<grid, 32>>>(g, p->d_ant, (double*)p->d_tab, p->d_D0);
  init_cis_kernel<<<1, 256>>>();  // fp64 phasor table (cis_rev) of the c128 kernels
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    free_plan(p);
    return fail(NF_ERR_CUDA, std::string("build_table: ") + cudaGetErrorString(e));
  }
  p->launches += 1;
  *out = p;
  return NF_OK;
}

int nf_plan_destroy(nf_plan* plan) {
  free_plan(plan);
  return NF_OK;
}

int nf_plan_info(const nf_plan* p, int64_t info[8]) {
  if (!p || !info) return fail(NF_ERR_ARG, "null argument");
  info[0] = p->nvox;
  info[1] = p->M;
  info[2] = p->g.ntiles;
  info[3] = p->g.Tg;
  info[4] = (int64_t)p->dev_bytes;
  info[5] = p->fwd_chunk;
  info[6] = p->dtype;
  info[7] = p->launches;
  return NF_OK;
}

int nf_batch_prepare(nf_plan* p, const int32_t* idx, int B, void* stream) {
  if (!p || !idx) return fail(NF_ERR_ARG, "null argument");
  if (B < 1) return fail(NF_ERR_ARG, "channel subset must be non-empty");
  if (B > p->max_batch) return fail(NF_ERR_ARG, "batch larger than the plan's max_batch");
  cudaStream_t st = (cudaStream_t)stream;
  const bool pdl = p->use_pdl;
  p->structured = false;
  const bool rx = ct_rxmajor(p, B);
  const KeyMap km = rx ? p->km_rx : p->km;
  CUDA_TRY(launch_k(pdl, mark_kernel, dim3((B + 255) / 256), dim3(256), 0, st, km, idx, B, p->d_pos_of_key));
  CUDA_TRY(launch_k(pdl, count_kernel, dim3(p->ksblocks), dim3(1024), 0, st, (const int*)p->d_pos_of_key, p->KS,
                    p->d_cnt));
  CUDA_TRY(launch_k(pdl, scan_kernel, dim3(1), dim3(1024), 0, st, p->d_cnt, p->ksblocks));
  CUDA_TRY(launch_k(pdl, compact_kernel, dim3(p->ksblocks), dim3(1024), 0, st, km, p->d_pos_of_key, p->KS,
                    (const int*)p->d_cnt, p->d_sm, p->d_spos, p->d_crec, p->d_sf, (const double*)p->d_kd));
  p->launches += 4;
  p->B = B;
  p->rxmajor = rx;
  return NF_OK;
}

int nf_batch_prepare_structured(nf_plan* p, const int32_t* fs, int nf, const int32_t* ts, int nt, const int32_t* rs,
                                int nr, void* stream) {
  if (!p || !fs || !ts || !rs) return fail(NF_ERR_ARG, "null argument");
  const int lim[3] = {p->g.F, p->g.T, p->g.R};
  const int cnt[3] = {nf, nt, nr};
  const int32_t* lists[3] = {fs, ts, rs};
  const char* names[3] = {"frequency", "tx", "rx"};
  for (int k = 0; k < 3; ++k) {
    if (cnt[k] < 1 || cnt[k] > lim[k])
      return fail(NF_ERR_ARG, std::string(names[k]) + " count must be in [1, " + std::to_string(lim[k]) + "]");
    for (int i = 0; i < cnt[k]; ++i) {
      if (lists[k][i] < 0 || lists[k][i] >= lim[k])
        return fail(NF_ERR_ARG, std::string(names[k]) + " index out of range");
      if (i && lists[k][i] <= lists[k][i - 1])
        return fail(NF_ERR_ARG, std::string(names[k]) + " indices must be strictly increasing");
    }
  }
  const long long B = (long long)nf * nt * nr;
  if (B > p->max_batch) return fail(NF_ERR_ARG, "batch larger than the plan's max_batch");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int32_t> h((size_t)p->g.F + p->g.T + p->g.R, 0);
  std::memcpy(h.data(), fs, sizeof(int32_t) * nf);
  std::memcpy(h.data() + p->g.F, ts, sizeof(int32_t) * nt);
  std::memcpy(h.data() + p->g.F + p->g.T, rs, sizeof(int32_t) * nr);
  // pageable source: staged by the driver before the call returns, so h may go out of scope
  CUDA_TRY(cudaMemcpyAsync(p->d_struct, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice, st));
  p->snf = nf;
  p->snt = nt;
  p->snr = nr;
  const StructArgs sa = struct_args(p);
  struct_prep_kernel<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(sa, p->g.T, p->g.R, p->d_sm, p->d_spos, p->d_sf);
  CUDA_TRY(cudaGetLastError());
  p->launches += 1;
  p->B = (int)B;
  p->structured = true;
  return NF_OK;
}

int nf_forward(nf_plan* p, const void* s, void* y, void* stream) {
  if (!p || !s || !y) return fail(NF_ERR_ARG, "null argument");
  if (p->B < 1) return fail(NF_ERR_STATE, "no batch staged (call nf_batch_prepare first)");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->structured && p->dtype == NF_C64 && use_tc_struct(p, true)) return launch_forward_tc(p, s, y, st);
  if (p->structured)
    return p->dtype == NF_C64 ? launch_forward_struct<float>(p, s, y, st) : launch_forward_struct<double>(p, s, y, st);
  return p->dtype == NF_C64 ? launch_forward<float>(p, s, y, st) : launch_forward<double>(p, s, y, st);
}

int nf_comm_create(nf_plan* p, int rank, int world, void* handle_out) {
  if (!p || !handle_out) return fail(NF_ERR_ARG, "null argument");
  if (world < 1 || world > PEER_MAX) return fail(NF_ERR_ARG, "world must be in [1, 8]");
  if (rank < 0 || rank >= world) return fail(NF_ERR_ARG, "rank out of range");
  if (p->comm_buf) return fail(NF_ERR_STATE, "communicator already created for this plan");
  p->comm_world = world;
  p->comm_rank = rank;
  p->comm_cap = p->max_batch;
  p->comm_nblk = (p->max_batch + 255) / 256;  // one flag/epoch slot per 256 channels of the batch
  const size_t bytes = comm_recv_bytes(p) + (size_t)world * p->comm_nblk * sizeof(unsigned long long);
  CUDA_TRY(cudaMalloc(&p->comm_buf, bytes));
  CUDA_TRY(cudaMemset(p->comm_buf, 0, bytes));
  CUDA_TRY(cudaMalloc((void**)&p->d_epoch, p->comm_nblk * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemset(p->d_epoch, 0, p->comm_nblk * sizeof(unsigned long long)));
  CUDA_TRY(cudaMalloc((void**)&p->d_comm_err, sizeof(int)));
  CUDA_TRY(cudaMemset(p->d_comm_err, 0, sizeof(int)));
  p->dev_bytes += bytes + p->comm_nblk * sizeof(unsigned long long) + sizeof(int);
  CUDA_TRY(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, p->comm_buf));
  static_assert(sizeof(cudaIpcMemHandle_t) == NF_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, NF_IPC_HANDLE_BYTES);
  p->comm_peer[rank] = p->comm_buf;
  return NF_OK;
}

int nf_comm_connect(nf_plan* p, const void* handles) {
  if (!p || !handles) return fail(NF_ERR_ARG, "null argument");
  if (!p->comm_buf) return fail(NF_ERR_STATE, "nf_comm_create first");
  if (p->comm_connected) return fail(NF_ERR_STATE, "communicator already connected");
  for (int q = 0; q < p->comm_world; ++q) {
    if (q == p->comm_rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const char*)handles + (size_t)q * NF_IPC_HANDLE_BYTES, NF_IPC_HANDLE_BYTES);
    CUDA_TRY(cudaIpcOpenMemHandle(&p->comm_peer[q], h, cudaIpcMemLazyEnablePeerAccess));
  }
  p->comm_connected = true;
  return NF_OK;
}

int nf_forward_allreduce(nf_plan* p, const void* s, void* y, void* stream) {
  if (!p || !s || !y) return fail(NF_ERR_ARG, "null argument");
  if (!p->comm_connected) return fail(NF_ERR_STATE, "peer all-reduce not connected (nf_comm_create/nf_comm_connect)");
  p->comm_active = true;
  p->comm_fused = false;
  int rc = nf_forward(p, s, y, stream);
  p->comm_active = false;
  if (rc == NF_OK && !p->comm_fused) {  // structured batches: one-shot peer all-reduce of the finished y
    const int nblk = (p->B + 255) / 256;
    const PeerArgs pa = peer_args(p, 0, nullptr, y);
    cudaError_t e = p->dtype == NF_C64
                        ? launch_k(false, fwd_reduce2_peer_kernel<float, true>, dim3(nblk, 1), dim3(256), 0,
                                   (cudaStream_t)stream, pa, p->B, 0, 0, (const int*)nullptr, (const int*)nullptr,
                                   (const double*)nullptr)
                        : launch_k(false, fwd_reduce2_peer_kernel<double, true>, dim3(nblk, 1), dim3(256), 0,
                                   (cudaStream_t)stream, pa, p->B, 0, 0, (const int*)nullptr, (const int*)nullptr,
                                   (const double*)nullptr);
    if (e != cudaSuccess) return fail(NF_ERR_CUDA, std::string("peer all-reduce: ") + cudaGetErrorString(e));
    p->launches += 1;
  }
  return rc;
}

int nf_comm_status(nf_plan* p, int* timed_out) {
  if (!p || !timed_out) return fail(NF_ERR_ARG, "null argument");
  *timed_out = 0;
  if (!p->d_comm_err) return NF_OK;
  CUDA_TRY(cudaMemcpy(timed_out, p->d_comm_err, sizeof(int), cudaMemcpyDeviceToHost));
  return NF_OK;
}

int nf_comm_emulate(int dtype, int world, int span, int nseg, int epochs, const double* tmp_host,
                    const int* sf_host, const int* spos_host, const double* pulse_host, int n_f, double* y_host) {
  if (!tmp_host || !sf_host || !spos_host || !pulse_host || !y_host) return fail(NF_ERR_ARG, "null argument");
  if (world < 1 || world > PEER_MAX || span < 1 || nseg < 0 || epochs < 1 || n_f < 1)
    return fail(NF_ERR_ARG, "bad sizes");
  if (dtype != NF_C64 && dtype != NF_C128) return fail(NF_ERR_ARG, "dtype must be NF_C64 or NF_C128");
  const int nblk = (span + 255) / 256;
  const size_t rs = dtype == NF_C64 ? sizeof(float) : sizeof(double);
  const size_t recv_b = (size_t)2 * world * span * sizeof(double2), flag_b = (size_t)world * nblk * 8;
  std::vector<void*> bufs;
  auto dmal = [&](size_t b) -> void* {
    void* q = nullptr;
    if (cudaMalloc(&q, b) != cudaSuccess) return nullptr;
    cudaMemset(q, 0, b);
    bufs.push_back(q);
    return q;
  };
  int rc = NF_OK;
  PeerArgs pa = {};
  pa.world = world;
  pa.rank0 = 0;
  pa.cap = span;
  pa.nblk_cap = nblk;
  pa.blk_base = 0;
  int *sf = (int*)dmal(span * sizeof(int)), *sp = (int*)dmal(span * sizeof(int));
  double* pulse = (double*)dmal(2 * n_f * sizeof(double));
  pa.err = (int*)dmal(sizeof(int));
  std::vector<double> tmpd((size_t)std::max(nseg, 1) * span * 2);
  for (int q = 0; q < world && rc == NF_OK; ++q) {
    char* b = (char*)dmal(recv_b + flag_b);
    pa.tmp[q] = (const double2*)dmal(tmpd.size() * sizeof(double));
    pa.y[q] = dmal(2 * span * rs);
    pa.epoch[q] = (unsigned long long*)dmal(nblk * 8);
    if (!b || !pa.tmp[q] || !pa.y[q] || !pa.epoch[q]) rc = fail(NF_ERR_CUDA, "cudaMalloc failed");
    pa.recv[q] = (double2*)b;
    pa.flag[q] = (unsigned long long*)(b + recv_b);
  }
  if (rc == NF_OK && (!sf || !sp || !pulse || !pa.err)) rc = fail(NF_ERR_CUDA, "cudaMalloc failed");
  if (rc == NF_OK) {
    cudaMemcpy(sf, sf_host, span * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(sp, spos_host, span * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(pulse, pulse_host, 2 * n_f * sizeof(double), cudaMemcpyHostToDevice);
  }
  std::vector<char> yh(2 * span * rs);
  for (int ep = 0; ep < epochs && rc == NF_OK; ++ep) {
    for (int q = 0; q < world; ++q) {
      const double* src = tmp_host + ((size_t)ep * world + q) * std::max(nseg, 1) * span * 2;
      if (nseg > 0) {
        cudaMemcpy((void*)pa.tmp[q], src, (size_t)nseg * span * 2 * sizeof(double), cudaMemcpyHostToDevice);
      } else {  // nseg = 0: the input is y itself (the one-shot all-reduce of a finished y)
        for (int i = 0; i < 2 * span; ++i) {
          if (dtype == NF_C64)
            ((float*)yh.data())[i] = (float)src[i];
          else
            ((double*)yh.data())[i] = src[i];
        }
        cudaMemcpy(pa.y[q], yh.data(), yh.size(), cudaMemcpyHostToDevice);
      }
    }
    // one cooperative launch holds every emulated rank's blocks, so all of them are co-resident
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk, world);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (nseg > 0)
      e = dtype == NF_C64 ? cudaLaunchKernelEx(&cfg, fwd_reduce2_peer_kernel<float, false>, pa, span, nseg, 0,
                                               (const int*)sf, (const int*)sp, (const double*)pulse)
                          : cudaLaunchKernelEx(&cfg, fwd_reduce2_peer_kernel<double, false>, pa, span, nseg, 0,
                                               (const int*)sf, (const int*)sp, (const double*)pulse);
    else
      e = dtype == NF_C64 ? cudaLaunchKernelEx(&cfg, fwd_reduce2_peer_kernel<float, true>, pa, span, 0, 0,
                                               (const int*)sf, (const int*)sp, (const double*)pulse)
                          : cudaLaunchKernelEx(&cfg, fwd_reduce2_peer_kernel<double, true>, pa, span, 0, 0,
                                               (const int*)sf, (const int*)sp, (const double*)pulse);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      rc = fail(NF_ERR_CUDA, std::string("peer emulation: ") + cudaGetErrorString(e));
      break;
    }
    int err = 0;
    cudaMemcpy(&err, pa.err, sizeof(int), cudaMemcpyDeviceToHost);
    if (err) {
      rc = fail(NF_ERR_STATE, "peer emulation: a flag wait timed out");
      break;
    }
    for (int q = 0; q < world; ++q) {
      cudaMemcpy(yh.data(), pa.y[q], yh.size(), cudaMemcpyDeviceToHost);
      double* out = y_host + ((size_t)ep * world + q) * span * 2;
      for (int i = 0; i < 2 * span; ++i)
        out[i] = dtype == NF_C64 ? (double)((const float*)yh.data())[i] : ((const double*)yh.data())[i];
    }
  }
  for (void* q : bufs) cudaFree(q);
  return rc;
}

int nf_adjoint(nf_plan* p, const void* r, const void* ymeas, void* g, double scale, void* stream) {
  if (!p || !r || !g) return fail(NF_ERR_ARG, "null argument");
  if (p->B < 1) return fail(NF_ERR_STATE, "no batch staged (call nf_batch_prepare first)");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->dtype == NF_C64)
    return launch_adjoint<float, false>(p, r, ymeas, g, scale, nullptr, nullptr, 0, 0, nullptr, st);
  return launch_adjoint<double, false>(p, r, ymeas, g, scale, nullptr, nullptr, 0, 0, nullptr, st);
}

int nf_adjoint_prox(nf_plan* p, const void* r, const void* ymeas, const void* s_in, void* s_out,
                    double eta_over_b, double alpha, double* stats, void* stream) {
  if (!p || !r || !s_in || !s_out || !stats) return fail(NF_ERR_ARG, "null argument");
  if (s_in == s_out) return fail(NF_ERR_ARG, "s_in and s_out must not alias");
  if (!(alpha >= 0) || !std::isfinite(alpha)) return fail(NF_ERR_ARG, "alpha must be >= 0");
  if (p->B < 1) return fail(NF_ERR_STATE, "no batch staged (call nf_batch_prepare first)");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->dtype == NF_C64)
    return launch_adjoint<float, true>(p, r, ymeas, nullptr, 0, s_in, s_out, eta_over_b, alpha, stats, st);
  return launch_adjoint<double, true>(p, r, ymeas, nullptr, 0, s_in, s_out, eta_over_b, alpha, stats, st);
}

int nf_spgm_loop(nf_plan* p, const int32_t* idx_table, int iters, uint64_t seed, uint64_t iter0, int batch,
                 const void* ymeas, void* s_a, void* s_b, double eta_over_b, double alpha, double tol,
                 double time_budget_s, double* records, int* state, void* stream) {
  if (!p || !ymeas || !s_a || !s_b || !records || !state) return fail(NF_ERR_ARG, "null argument");
  if (s_a == s_b) return fail(NF_ERR_ARG, "s_a and s_b must not alias");
  if (iters < 1) return fail(NF_ERR_ARG, "iters must be >= 1");
  if (batch < 1 || batch > p->M) return fail(NF_ERR_ARG, "batch must be in [1, M]");
  if (!(alpha >= 0) || !std::isfinite(alpha)) return fail(NF_ERR_ARG, "alpha must be >= 0");
  if (batch > p->max_batch || batch > p->fwd_chunk || batch > LOOP_SORT_MAX)
    return fail(NF_ERR_STATE, "persistent loop: batch exceeds the plan's single forward window or the sort size");
  const long long budget = time_budget_s >= 0 && std::isfinite(time_budget_s) ? (long long)(time_budget_s * 1e9) : -1;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->dtype == NF_C64)
    return launch_spgm_loop<float>(p, idx_table, iters, seed, iter0, batch, ymeas, s_a, s_b, eta_over_b, alpha, tol,
                                   budget, records, state, st);
  return launch_spgm_loop<double>(p, idx_table, iters, seed, iter0, batch, ymeas, s_a, s_b, eta_over_b, alpha, tol,
                                  budget, records, state, st);
}

int nf_spgm_loop_chained(nf_plan* p, const int32_t* idx_table, int iters, uint64_t seed, uint64_t iter0, int batch,
                         const void* ymeas, void* s_a, void* s_b, double eta_over_b, double alpha, double tol,
                         double time_budget_s, double* records, int* state, const int* prev_state, void* stream) {
  if (!p) return fail(NF_ERR_ARG, "null argument");
  if (prev_state && prev_state == state) return fail(NF_ERR_ARG, "prev_state and state must not alias");
  p->loop_prev = prev_state;
  p->loop_fold = 1;
  const int rc = nf_spgm_loop(p, idx_table, iters, seed, iter0, batch, ymeas, s_a, s_b, eta_over_b, alpha, tol,
                              time_budget_s, records, state, stream);
  p->loop_prev = nullptr;
  p->loop_fold = 0;
  return rc;
}

// diagnostics: copy the persistent loop's phase time stamps of its last launch (NFGPU_LOOP_PROFILE) to the host
int nf_loop_profile(nf_plan* p, unsigned long long* host, int iters) {
  if (!p || !host) return fail(NF_ERR_ARG, "null argument");
  // iters: time stamps to copy (K * LOOP_PROF, plus K * 2 * LOOP_PROF_CTA with NFGPU_LOOP_PROFILE=2)
  if (!p->d_loop_prof || (size_t)iters > p->loop_prof_elems) return fail(NF_ERR_STATE, "no loop profile");
  CUDA_TRY(cudaMemcpy(host, p->d_loop_prof, (size_t)iters * 8, cudaMemcpyDeviceToHost));
  return NF_OK;
}

int nf_sample_structured(nf_plan* p, uint64_t seed, uint64_t iter, int nf, int nt, int nr, int32_t* lists,
                         void* stream) {
  if (!p) return fail(NF_ERR_ARG, "null argument");
  if (nf < 1 || nf > p->g.F || nt < 1 || nt > p->g.T || nr < 1 || nr > p->g.R)
    return fail(NF_ERR_ARG, "composition must satisfy 1 <= n_f <= F, 1 <= n_tx <= T, 1 <= n_rx <= R");
  const long long B = (long long)nf * nt * nr;
  if (B > p->max_batch) return fail(NF_ERR_ARG, "batch larger than the plan's max_batch");
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev = iter == NF_ITER_DEVICE;
  struct_sample_kernel<<<1, 256, 0, st>>>(seed, iter, dev ? p->d_iter : nullptr, p->g.F, p->g.T, p->g.R, nf, nt, nr,
                                          p->d_struct);
  CUDA_TRY(cudaGetLastError());
  p->snf = nf;
  p->snt = nt;
  p->snr = nr;
  const StructArgs sa = struct_args(p);
  struct_prep_kernel<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(sa, p->g.T, p->g.R, p->d_sm, p->d_spos, p->d_sf);
  CUDA_TRY(cudaGetLastError());
  p->launches += 2;
  if (lists) {  // copy of the drawn lists, [fs | ts | rs]
    CUDA_TRY(cudaMemcpyAsync(lists, sa.fs, sizeof(int) * nf, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(lists + nf, sa.ts, sizeof(int) * nt, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(lists + nf + nt, sa.rs, sizeof(int) * nr, cudaMemcpyDeviceToDevice, st));
  }
  p->B = (int)B;
  p->structured = true;
  return NF_OK;
}

int nf_sample_flat(nf_plan* p, uint64_t seed, uint64_t iter, int B, int32_t* idx, void* stream) {
  if (!p || !idx) return fail(NF_ERR_ARG, "null argument");
  if (B < 1 || B > p->M) return fail(NF_ERR_ARG, "batch must be in [1, M]");
  int bits = 2;
  while ((1LL << bits) < p->M) bits += 2;
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev = iter == NF_ITER_DEVICE;
  CUDA_TRY(launch_k(p->use_pdl, sample_kernel, dim3((B + 255) / 256), dim3(256), 0, st, seed, iter,
                    (const unsigned long long*)(dev ? p->d_iter : nullptr), bits / 2, p->M, B, idx));
  p->launches += 1;
  if (dev) {
    CUDA_TRY(launch_k(p->use_pdl, bump_kernel, dim3(1), dim3(1), 0, st, p->d_iter));
    p->launches += 1;
  }
  return NF_OK;
}

int nf_plan_set_iter(nf_plan* p, uint64_t iter, void* stream) {
  if (!p) return fail(NF_ERR_ARG, "null argument");
  set_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(p->d_iter, (unsigned long long)iter);
  CUDA_TRY(cudaGetLastError());
  p->launches += 1;
  return NF_OK;
}

int nf_soft_threshold(int dtype, const void* v, void* out, int64_t n, double alpha, void* stream) {
  if (!v || !out) return fail(NF_ERR_ARG, "null argument");
  if (dtype != NF_C64 && dtype != NF_C128) return fail(NF_ERR_ARG, "bad dtype");
  if (!(alpha >= 0) || !std::isfinite(alpha)) return fail(NF_ERR_ARG, "alpha must be >= 0");
  if (n <= 0) return NF_OK;
  const int64_t blocks = (n + 255) / 256;
  if (dtype == NF_C64)
    soft_threshold_kernel<float><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((const float*)v, (float*)out, n,
                                                                                     alpha);
  else
    soft_threshold_kernel<double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((const double*)v,
                                                                                      (double*)out, n, alpha);
  CUDA_TRY(cudaGetLastError());
  return NF_OK;
}

int nf_magnitude_change(int dtype, const void* a, const void* b, int64_t n, double* stats, void* stream) {
  if (!a || !b || !stats) return fail(NF_ERR_ARG, "null argument");
  if (dtype != NF_C64 && dtype != NF_C128) return fail(NF_ERR_ARG, "bad dtype");
  if (n < 0) return fail(NF_ERR_ARG, "n must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == NF_C64)
    magchange_kernel<float><<<1, 1024, 0, st>>>((const float*)a, (const float*)b, n, stats);
  else
    magchange_kernel<double><<<1, 1024, 0, st>>>((const double*)a, (const double*)b, n, stats);
  CUDA_TRY(cudaGetLastError());
  return NF_OK;
}

}  // extern "C"
