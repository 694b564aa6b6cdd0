// nfgpu.cu — B200 (sm_100a) kernels and C ABI for the SPGM hot path of the
// near-field MIMO imaging reference `nfmimo` (arXiv 2509.00774).
//
// The reference (pkg/src/nfmimo/forward.py:183-336) caches F×(T+R)×N complex128
// phasor tables. Each forward/adjoint is then elementwise products plus BLAS dots.
// Here nothing frequency-dependent is stored. Every operator entry
//     A[m,n] = p_f exp(-j 2π f (dT+dR)/c) / (4π dT dR)            (forward.py:142-155)
// is regenerated in registers from a frequency-free per-(antenna, voxel)
// distance table (8 B per pair in c64) and two MUFU ops (sin, cos).
//
// Work decomposition:
//   * voxels are cut into warp tiles of 8×4×4 = 128 voxels. Lane L owns 4 voxels
//     that are consecutive in x (coalesced s loads, conflict-free smem rows).
//   * each tile has an fp64 anchor (its centre). The table stores
//     δ = d − D0(tile, antenna) in fp32, plus 1/d. The per-(channel, tile) phase
//     offset frac(f/c·(D0_T+D0_R)) is computed once in fp64. Per entry the
//     phase is x = base + (f/c)·(δT+δR) with |x| <~ 8 rev. It is reduced to
//     [-½,½] and fed to __sincosf. This keeps ~1e-6 rad accuracy at phases of ~2e3 rad.
//   * the channel batch is sorted on the device by (tx-group, rx, tx, f).
//     A warp keeps the rx-side table entries for the current rx run in registers.
//     The tx-side entries of the current tx group sit in shared memory, so each
//     entry costs one conflict-free 16-byte shared load per 4 voxels.
//   * forward: per-channel lane partials → warp transpose-reduce through smem →
//     CTA combine → deterministic cross-CTA column reduce (fp64) in a second kernel.
//   * adjoint: a warp owns its tile for the whole batch (no reduction across warps).
//     The complex soft-threshold prox (solver.py:228-241) and the termination
//     statistics (solver.py:244-251) run in the epilogue.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nfgpu.h"

namespace {

constexpr int V = 4;            // voxels per lane
constexpr int TILE_X = 8, TILE_Y = 4, TILE_Z = 4;
constexpr int TILE = TILE_X * TILE_Y * TILE_Z;  // 128 = 32 lanes × V
constexpr int FWD_WARPS = 4;
constexpr int ADJ_WARPS = 4;
constexpr int TG_MAX_F = 12;    // tx per smem group (c64): 12 KB smem per warp
constexpr int TG_MAX_D = 6;     // tx per smem group (c128): 12 KB smem per warp
constexpr double PI = 3.14159265358979323846;

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

// ------------------------------------------------------------------ phasor
// cos/sin(2π·rev) of rev = base + k·dsum with the revolution count reduced to [-½, ½]
// before the MUFU (magic-number round-to-nearest, exact for |x| < 2^22).
__device__ __forceinline__ void phasor(float k, float base, float dsum, float& c, float& s) {
  float x = fmaf(k, dsum, base);
  float u = x + 12582912.0f;
  float r = u - 12582912.0f;
  float fr = x - r;
  __sincosf(fr * 6.28318530717958647692f, &s, &c);
}
__device__ __forceinline__ void phasor(double k, double base, double dsum, double& c, double& s) {
  double x = fma(k, dsum, base);
  double fr = x - rint(x);
  sincospi(2.0 * fr, &s, &c);
}

template <typename Real>
struct Vec4T;
template <>
struct Vec4T<float> {
  using T = float4;
};
template <>
struct Vec4T<double> {
  using T = double4;
};

template <typename Real>
__device__ __forceinline__ void ld4(const Real* p, Real (&v)[4]) {
  using V4 = typename Vec4T<Real>::T;
  V4 q = *reinterpret_cast<const V4*>(p);
  v[0] = q.x;
  v[1] = q.y;
  v[2] = q.z;
  v[3] = q.w;
}

// ------------------------------------------------------------------ geometry
struct Geo {
  int T, R, A, F;
  int nx, ny, nzs, zb;  // slab: nzs planes starting at global plane zb
  int ntx, nty, ntz, ntiles;
  int Tg, ng;
  double corner[3], sp[3];
};

__device__ __forceinline__ void tile_coords(const Geo& g, int tile, int& tx, int& ty, int& tz) {
  tz = tile / (g.ntx * g.nty);
  int rem = tile - tz * g.ntx * g.nty;
  ty = rem / g.ntx;
  tx = rem - ty * g.ntx;
}

// lane L of tile (tx,ty,tz) owns voxels x = 8tx + 4(L&1) + v, y = 4ty + ((L>>1)&3), z = 4tz + (L>>3)
__device__ __forceinline__ void lane_voxel(const Geo& g, int tx, int ty, int tz, int L, int& x0, int& y,
                                           int& z) {
  x0 = tx * TILE_X + (L & 1) * V;
  y = ty * TILE_Y + ((L >> 1) & 3);
  z = tz * TILE_Z + (L >> 3);
}

// table[tile][a][2][32][4]: [0] = δ, [1] = 1/d for the lane's 4 voxels; D0[tile][a] fp64.
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
  lane_voxel(g, tx, ty, tz, L, x0, y, z);
  Real* out = tab + ((size_t)tile * g.A + a) * (2 * 32 * V);
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
    out[L * V + v] = dl;
    out[32 * V + L * V + v] = iv;
  }
}

// ------------------------------------------------------------------ batch prep
struct KeyMap {
  int T, R, F, Tg;
};
__device__ __forceinline__ int key_of(const KeyMap& k, int m) {
  const int TR = k.T * k.R;
  const int f = m / TR;
  const int rem = m - f * TR;
  const int t = rem / k.R;
  const int r = rem - t * k.R;
  const int tg = t / k.Tg, tl = t - tg * k.Tg;
  return ((tg * k.R + r) * k.Tg + tl) * k.F + f;
}
__device__ __forceinline__ int m_of_key(const KeyMap& k, int key, bool& ok) {
  const int f = key % k.F;
  int q = key / k.F;
  const int tl = q % k.Tg;
  q /= k.Tg;
  const int r = q % k.R;
  const int tg = q / k.R;
  const int t = tg * k.Tg + tl;
  ok = t < k.T;
  return r + k.R * (t + k.T * f);
}

__global__ void mark_kernel(KeyMap km, const int* __restrict__ idx, int B, int* __restrict__ pos_of_key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) pos_of_key[key_of(km, idx[i])] = i;
}

__device__ __forceinline__ int block_excl_scan_1024(int v, int* sh, int& total) {
  // 1024 threads; sh >= 32 ints
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
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

__global__ void __launch_bounds__(1024) count_kernel(const int* __restrict__ pos_of_key, int KS,
                                                      int* __restrict__ cnt) {
  __shared__ int sh[32];
  const int key = blockIdx.x * 1024 + threadIdx.x;
  const int f = (key < KS && pos_of_key[key] >= 0) ? 1 : 0;
  const int c = __syncthreads_count(f);
  (void)sh;
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) scan_kernel(int* __restrict__ cnt, int n) {
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

__global__ void __launch_bounds__(1024) compact_kernel(KeyMap km, int* __restrict__ pos_of_key, int KS,
                                                        const int* __restrict__ off, int* __restrict__ sm,
                                                        int* __restrict__ spos) {
  __shared__ int sh[32];
  const int key = blockIdx.x * 1024 + threadIdx.x;
  const int p = key < KS ? pos_of_key[key] : -1;
  int total;
  const int pre = block_excl_scan_1024(p >= 0 ? 1 : 0, sh, total);
  if (p >= 0) {
    bool ok;
    const int j = off[blockIdx.x] + pre;
    sm[j] = m_of_key(km, key, ok);
    spos[j] = p;
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
    const uint32_t k = (uint32_t)(key >> (round & 1 ? 32 : 0)) ^ (0x9e3779b9u * (round + 1));
    const uint32_t f = hash32(r ^ k) & mask;
    const uint32_t nl = r;
    r = l ^ f;
    l = nl;
  }
  return (l << hb) | r;
}
__global__ void sample_kernel(uint64_t key, int hb, int M, int B, int* __restrict__ idx) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B) return;
  uint32_t x = (uint32_t)j;
  do {
    x = feistel(x, hb, key);
  } while (x >= (uint32_t)M);
  idx[j] = (int)x;
}

// ------------------------------------------------------------------ forward
template <typename Real>
struct FwdRec {
  Real k, base;
  int tl, r, tg, pad;
};

template <typename Real>
struct FwdArgs {
  Geo g;
  const Real* __restrict__ tab;
  const double* __restrict__ D0;
  const double* __restrict__ kd;
  const Real* __restrict__ kf;
  const Real* __restrict__ s;  // complex, slab-local flat order
  const int* __restrict__ sm;  // sorted channel ids
  int j0, j1;                  // sorted positions of this chunk
  int Q;                       // channel splits (gridDim.y)
  Real* __restrict__ partials;  // [gridDim.x][j1-j0] complex
};

template <typename Real>
__global__ void __launch_bounds__(FWD_WARPS * 32) fwd_kernel(FwdArgs<Real> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& g = a.g;
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int tile = blockIdx.x * FWD_WARPS + w;
  const bool tile_ok = tile < g.ntiles;
  const int per_t = g.Tg * 2 * 32 * V;  // Reals per warp tx-group buffer
  Real* tside = reinterpret_cast<Real*>(smem_raw) + (size_t)w * per_t;
  FwdRec<Real>* rec =
      reinterpret_cast<FwdRec<Real>*>(reinterpret_cast<Real*>(smem_raw) + (size_t)FWD_WARPS * per_t) +
      w * 32;
  Real* tb = reinterpret_cast<Real*>(reinterpret_cast<FwdRec<Real>*>(
                 reinterpret_cast<Real*>(smem_raw) + (size_t)FWD_WARPS * per_t) +
                                     FWD_WARPS * 32);
  Real* cbuf = tb + (size_t)FWD_WARPS * 32 * 33 * 2;  // [2][W][32] complex
  Real* mytb = tb + (size_t)w * 32 * 33 * 2;

  int tx = 0, ty = 0, tz = 0;
  if (tile_ok) tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(g, tx, ty, tz, L, x0, y, z);
  Real sr[V], si[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int x = x0 + v;
    const bool ok = tile_ok && x < g.nx && y < g.ny && z < g.nzs;
    const size_t n = ((size_t)z * g.ny + y) * g.nx + x;
    sr[v] = ok ? a.s[2 * n] : Real(0);
    si[v] = ok ? a.s[2 * n + 1] : Real(0);
  }

  const int span = a.j1 - a.j0;
  const int c0 = a.j0 + (int)(((long long)span * blockIdx.y) / a.Q);
  const int c1 = a.j0 + (int)(((long long)span * (blockIdx.y + 1)) / a.Q);
  const size_t prow = (size_t)blockIdx.x * span;
  const Real* tabt = a.tab + (size_t)(tile_ok ? tile : 0) * g.A * (2 * 32 * V);

  int cur_tg = -1, cur_r = -1;
  Real dR[V], iR[V], shr[V], shi[V];
#pragma unroll
  for (int v = 0; v < V; ++v) dR[v] = iR[v] = shr[v] = shi[v] = 0;
  int par = 0;
  for (int jb = c0; jb < c1; jb += 32) {
    const int nb = min(32, c1 - jb);
    if (L < nb) {
      const int m = a.sm[jb + L];
      const int TR = g.T * g.R;
      const int f = m / TR, rem = m - f * TR, t = rem / g.R, r = rem - t * g.R;
      const int tg = t / g.Tg;
      double base = 0;
      if (tile_ok) {
        const double D = a.D0[(size_t)tile * g.A + t] + a.D0[(size_t)tile * g.A + g.T + r];
        const double xx = a.kd[f] * D;
        base = xx - rint(xx);
      }
      FwdRec<Real> q;
      q.k = a.kf[f];
      q.base = (Real)base;
      q.tl = t - tg * g.Tg;
      q.r = r;
      q.tg = tg;
      q.pad = 0;
      rec[L] = q;
    }
    __syncwarp();
    for (int c = 0; c < nb; ++c) {
      const FwdRec<Real> q = rec[c];
      if (q.tg != cur_tg) {
        __syncwarp();
        const int ta = q.tg * g.Tg;
        const int nt = min(g.Tg, g.T - ta);
        const Real* src = tabt + (size_t)ta * (2 * 32 * V);
        for (int i = L; i < nt * 2 * 32; i += 32) {
          Real v4[4];
          ld4(src + (size_t)i * V, v4);
#pragma unroll
          for (int v = 0; v < V; ++v) tside[i * V + v] = v4[v];
        }
        __syncwarp();
        cur_tg = q.tg;
      }
      if (q.r != cur_r) {
        const Real* src = tabt + (size_t)(g.T + q.r) * (2 * 32 * V);
        ld4(src + L * V, dR);
        ld4(src + 32 * V + L * V, iR);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          shr[v] = iR[v] * sr[v];
          shi[v] = iR[v] * si[v];
        }
        cur_r = q.r;
      }
      Real dT[V], iT[V];
      ld4(tside + (size_t)q.tl * (2 * 32 * V) + L * V, dT);
      ld4(tside + (size_t)q.tl * (2 * 32 * V) + 32 * V + L * V, iT);
      Real pr = 0, pi = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        Real cs, sn;
        phasor(q.k, q.base, dT[v] + dR[v], cs, sn);
        const Real aa = iT[v] * cs, bb = iT[v] * sn;
        pr += aa * shr[v] + bb * shi[v];
        pi += aa * shi[v] - bb * shr[v];
      }
      mytb[(c * 33 + L) * 2] = pr;
      mytb[(c * 33 + L) * 2 + 1] = pi;
    }
    __syncwarp();
    Real Sr = 0, Si = 0;
    if (L < nb) {
#pragma unroll 8
      for (int l = 0; l < 32; ++l) {
        Sr += mytb[(L * 33 + l) * 2];
        Si += mytb[(L * 33 + l) * 2 + 1];
      }
    }
    cbuf[((par * FWD_WARPS + w) * 32 + L) * 2] = Sr;
    cbuf[((par * FWD_WARPS + w) * 32 + L) * 2 + 1] = Si;
    __syncthreads();
    if (w == 0 && L < nb) {
      Real tr = 0, ti = 0;
#pragma unroll
      for (int ww = 0; ww < FWD_WARPS; ++ww) {
        tr += cbuf[((par * FWD_WARPS + ww) * 32 + L) * 2];
        ti += cbuf[((par * FWD_WARPS + ww) * 32 + L) * 2 + 1];
      }
      const size_t o = prow + (jb + L - a.j0);
      a.partials[2 * o] = tr;
      a.partials[2 * o + 1] = ti;
    }
    par ^= 1;
  }
}

// y[spos[j]] = p_f/(4π) Σ_x partials[x][j]  (fp64 accumulation, fixed order)
template <typename Real>
__global__ void fwd_reduce_kernel(const Real* __restrict__ partials, int nx_blocks, int span, int j0,
                                  const int* __restrict__ sm, const int* __restrict__ spos, int TR,
                                  const double* __restrict__ pulse, Real* __restrict__ y) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= span) return;
  double sr = 0, si = 0;
  for (int x = 0; x < nx_blocks; ++x) {
    const size_t o = (size_t)x * span + j;
    sr += (double)partials[2 * o];
    si += (double)partials[2 * o + 1];
  }
  const int m = sm[j0 + j];
  const int f = m / TR;
  const double pr = pulse[2 * f] / (4.0 * PI), pim = pulse[2 * f + 1] / (4.0 * PI);
  const int k = spos[j0 + j];
  y[2 * (size_t)k] = (Real)(pr * sr - pim * si);
  y[2 * (size_t)k + 1] = (Real)(pr * si + pim * sr);
}

// ------------------------------------------------------------------ adjoint (+prox)
template <typename Real>
struct AdjRec {
  Real k, base, wr, wi;
  int tl, r, tg, pad;
};

template <typename Real>
struct AdjArgs {
  Geo g;
  const Real* __restrict__ tab;
  const double* __restrict__ D0;
  const double* __restrict__ kd;
  const Real* __restrict__ kf;
  const double* __restrict__ pulse;
  const int* __restrict__ sm;
  const int* __restrict__ spos;
  int B;
  const Real* __restrict__ r;      // subset order
  const Real* __restrict__ ymeas;  // full M or null
  // plain adjoint
  Real* __restrict__ gout;
  double scale;
  // prox
  const Real* __restrict__ s_in;
  Real* __restrict__ s_out;
  double eta_over_b, alpha;
  double* __restrict__ stat_part;  // [ntiles][4]
};

template <typename Real, bool PROX>
__global__ void __launch_bounds__(ADJ_WARPS * 32) adj_kernel(AdjArgs<Real> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geo& g = a.g;
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  const int tile = blockIdx.x * ADJ_WARPS + w;
  if (tile >= g.ntiles) return;  // warps are independent: no block barriers below
  const int per_t = g.Tg * 2 * 32 * V;
  Real* tside = reinterpret_cast<Real*>(smem_raw) + (size_t)w * per_t;
  AdjRec<Real>* rec =
      reinterpret_cast<AdjRec<Real>*>(reinterpret_cast<Real*>(smem_raw) + (size_t)ADJ_WARPS * per_t) +
      w * 32;
  int tx, ty, tz;
  tile_coords(g, tile, tx, ty, tz);
  int x0, y, z;
  lane_voxel(g, tx, ty, tz, L, x0, y, z);
  const Real* tabt = a.tab + (size_t)tile * g.A * (2 * 32 * V);
  const int TR = g.T * g.R;

  Real gr[V], gi[V], hr[V], hi[V], dR[V], iR[V];
#pragma unroll
  for (int v = 0; v < V; ++v) gr[v] = gi[v] = hr[v] = hi[v] = dR[v] = iR[v] = 0;
  int cur_tg = -1, cur_r = -1;
  double dfid = 0;  // Σ |r - y|^2 over the batch (tile 0 only)

  for (int jb = 0; jb < a.B; jb += 32) {
    const int nb = min(32, a.B - jb);
    __syncwarp();
    if (L < nb) {
      const int m = a.sm[jb + L];
      const int f = m / TR, rem = m - f * TR, t = rem / g.R, r = rem - t * g.R;
      const int tg = t / g.Tg;
      const double D = a.D0[(size_t)tile * g.A + t] + a.D0[(size_t)tile * g.A + g.T + r];
      const double xx = a.kd[f] * D;
      const int k = a.spos[jb + L];
      double rr = (double)a.r[2 * (size_t)k], ri = (double)a.r[2 * (size_t)k + 1];
      if (a.ymeas) {
        rr -= (double)a.ymeas[2 * (size_t)m];
        ri -= (double)a.ymeas[2 * (size_t)m + 1];
      }
      if (tile == 0) dfid += rr * rr + ri * ri;
      // w = conj(p_f)/(4π) · r
      const double pr = a.pulse[2 * f] / (4.0 * PI), pim = -a.pulse[2 * f + 1] / (4.0 * PI);
      AdjRec<Real> q;
      q.k = a.kf[f];
      q.base = (Real)(xx - rint(xx));
      q.wr = (Real)(pr * rr - pim * ri);
      q.wi = (Real)(pr * ri + pim * rr);
      q.tl = t - tg * g.Tg;
      q.r = r;
      q.tg = tg;
      q.pad = 0;
      rec[L] = q;
    }
    __syncwarp();
    for (int c = 0; c < nb; ++c) {
      const AdjRec<Real> q = rec[c];
      if (q.tg != cur_tg) {
        __syncwarp();
        const int ta = q.tg * g.Tg;
        const int nt = min(g.Tg, g.T - ta);
        const Real* src = tabt + (size_t)ta * (2 * 32 * V);
        for (int i = L; i < nt * 2 * 32; i += 32) {
          Real v4[4];
          ld4(src + (size_t)i * V, v4);
#pragma unroll
          for (int v = 0; v < V; ++v) tside[i * V + v] = v4[v];
        }
        __syncwarp();
        cur_tg = q.tg;
      }
      if (q.r != cur_r) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          gr[v] += iR[v] * hr[v];
          gi[v] += iR[v] * hi[v];
          hr[v] = hi[v] = 0;
        }
        const Real* src = tabt + (size_t)(g.T + q.r) * (2 * 32 * V);
        ld4(src + L * V, dR);
        ld4(src + 32 * V + L * V, iR);
        cur_r = q.r;
      }
      Real dT[V], iT[V];
      ld4(tside + (size_t)q.tl * (2 * 32 * V) + L * V, dT);
      ld4(tside + (size_t)q.tl * (2 * 32 * V) + 32 * V + L * V, iT);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        Real cs, sn;
        phasor(q.k, q.base, dT[v] + dR[v], cs, sn);
        const Real aa = iT[v] * cs, bb = iT[v] * sn;
        hr[v] += aa * q.wr - bb * q.wi;
        hi[v] += aa * q.wi + bb * q.wr;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    gr[v] += iR[v] * hr[v];
    gi[v] += iR[v] * hi[v];
  }

  double st0 = 0, st1 = 0, st3 = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int x = x0 + v;
    if (!(x < g.nx && y < g.ny && z < g.nzs)) continue;
    const size_t n = ((size_t)z * g.ny + y) * g.nx + x;
    if (!PROX) {
      a.gout[2 * n] = (Real)(a.scale * gr[v]);
      a.gout[2 * n + 1] = (Real)(a.scale * gi[v]);
    } else {
      const Real s_r = a.s_in[2 * n], s_i = a.s_in[2 * n + 1];
      const Real ur = s_r - (Real)a.eta_over_b * gr[v];
      const Real ui = s_i - (Real)a.eta_over_b * gi[v];
      const Real mag = sqrt(ur * ur + ui * ui);
      const Real al = (Real)a.alpha;
      const Real sc = mag > al ? (mag - al) / mag : Real(0);
      const Real o_r = ur * sc, o_i = ui * sc;
      a.s_out[2 * n] = o_r;
      a.s_out[2 * n + 1] = o_i;
      const double m0 = sqrt((double)s_r * s_r + (double)s_i * s_i);
      const double m1 = sqrt((double)o_r * o_r + (double)o_i * o_i);
      st0 += m0 * m0;
      st1 += (m1 - m0) * (m1 - m0);
      st3 += m1;
    }
  }
  if (PROX) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st0 += __shfl_xor_sync(0xffffffffu, st0, o);
      st1 += __shfl_xor_sync(0xffffffffu, st1, o);
      st3 += __shfl_xor_sync(0xffffffffu, st3, o);
      dfid += __shfl_xor_sync(0xffffffffu, dfid, o);
    }
    if (L == 0) {
      a.stat_part[(size_t)tile * 4 + 0] = st0;
      a.stat_part[(size_t)tile * 4 + 1] = st1;
      a.stat_part[(size_t)tile * 4 + 2] = 0.5 * dfid;
      a.stat_part[(size_t)tile * 4 + 3] = st3;
    }
  }
}

// stats[q] = Σ_tile part[tile][q] in a fixed order (deterministic)
__global__ void __launch_bounds__(256) stats_reduce_kernel(const double* __restrict__ part, int n,
                                                           double* __restrict__ out) {
  __shared__ double sh[4][256];
  double acc[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < n; i += 256)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += part[(size_t)i * 4 + q];
#pragma unroll
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 4) out[threadIdx.x] = sh[threadIdx.x][0];
}

// ------------------------------------------------------------------ elementwise utilities
template <typename Real>
__global__ void soft_threshold_kernel(const Real* __restrict__ v, Real* __restrict__ out, int64_t n,
                                      double alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double vr = v[2 * i], vi = v[2 * i + 1];
  const double mag = sqrt(vr * vr + vi * vi);
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
    const double ma = sqrt((double)a[2 * i] * a[2 * i] + (double)a[2 * i + 1] * a[2 * i + 1]);
    const double mb = sqrt((double)b[2 * i] * b[2 * i] + (double)b[2 * i + 1] * b[2 * i + 1]);
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
  int fwd_chunk;
  size_t dev_bytes = 0;
  int64_t launches = 0;
  int KS, ksblocks;
  KeyMap km;
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
  void* d_partials = nullptr;
  double* d_stat_part = nullptr;
};

namespace {

template <typename T>
int dalloc(nf_plan* p, T** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc((void**)ptr, bytes);
  if (e != cudaSuccess)
    return fail(NF_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  p->dev_bytes += bytes;
  return NF_OK;
}

void free_plan(nf_plan* p) {
  if (!p) return;
  cudaFree(p->d_ant);
  cudaFree(p->d_kd);
  cudaFree(p->d_kf);
  cudaFree(p->d_pulse);
  cudaFree(p->d_tab);
  cudaFree(p->d_D0);
  cudaFree(p->d_pos_of_key);
  cudaFree(p->d_cnt);
  cudaFree(p->d_sm);
  cudaFree(p->d_spos);
  cudaFree(p->d_partials);
  cudaFree(p->d_stat_part);
  delete p;
}

size_t real_size(const nf_plan* p) { return p->dtype == NF_C64 ? sizeof(float) : sizeof(double); }

size_t fwd_smem(const nf_plan* p) {
  const size_t rs = real_size(p);
  const size_t recsz = p->dtype == NF_C64 ? sizeof(FwdRec<float>) : sizeof(FwdRec<double>);
  return (size_t)FWD_WARPS * p->g.Tg * 2 * 32 * V * rs + (size_t)FWD_WARPS * 32 * recsz +
         (size_t)FWD_WARPS * 32 * 33 * 2 * rs + (size_t)2 * FWD_WARPS * 32 * 2 * rs;
}
size_t adj_smem(const nf_plan* p) {
  const size_t rs = real_size(p);
  const size_t recsz = p->dtype == NF_C64 ? sizeof(AdjRec<float>) : sizeof(AdjRec<double>);
  return (size_t)ADJ_WARPS * p->g.Tg * 2 * 32 * V * rs + (size_t)ADJ_WARPS * 32 * recsz;
}

int channel_splits(const nf_plan* p, int span) {
  // enough CTAs for ~8 waves of 2 CTAs/SM on 148 SMs; ≥ 32 channels per split
  const long long target = 148LL * 2 * 8;
  long long q = (target + p->fwd_gridx - 1) / p->fwd_gridx;
  long long qmax = std::max(1, span / 32);
  if (q > qmax) q = qmax;
  if (q < 1) q = 1;
  return (int)q;
}

template <typename Real>
int launch_forward(nf_plan* p, const void* s, void* y, cudaStream_t st) {
  const size_t sm = fwd_smem(p);
  CUDA_TRY(cudaFuncSetAttribute(fwd_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  for (int j0 = 0; j0 < p->B; j0 += p->fwd_chunk) {
    const int j1 = std::min(p->B, j0 + p->fwd_chunk);
    FwdArgs<Real> a;
    a.g = p->g;
    a.tab = (const Real*)p->d_tab;
    a.D0 = p->d_D0;
    a.kd = p->d_kd;
    a.kf = (const Real*)p->d_kf;
    a.s = (const Real*)s;
    a.sm = p->d_sm;
    a.j0 = j0;
    a.j1 = j1;
    a.Q = channel_splits(p, j1 - j0);
    a.partials = (Real*)p->d_partials;
    dim3 grid(p->fwd_gridx, a.Q);
    fwd_kernel<Real><<<grid, FWD_WARPS * 32, sm, st>>>(a);
    CUDA_TRY(cudaGetLastError());
    const int span = j1 - j0;
    fwd_reduce_kernel<Real><<<(span + 255) / 256, 256, 0, st>>>(
        (const Real*)p->d_partials, p->fwd_gridx, span, j0, p->d_sm, p->d_spos, p->g.T * p->g.R, p->d_pulse,
        (Real*)y);
    CUDA_TRY(cudaGetLastError());
    p->launches += 2;
  }
  return NF_OK;
}

template <typename Real, bool PROX>
int launch_adjoint(nf_plan* p, const void* r, const void* ymeas, void* gout, double scale, const void* s_in,
                   void* s_out, double eta_over_b, double alpha, double* stats, cudaStream_t st) {
  const size_t sm = adj_smem(p);
  CUDA_TRY(cudaFuncSetAttribute(adj_kernel<Real, PROX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  AdjArgs<Real> a;
  a.g = p->g;
  a.tab = (const Real*)p->d_tab;
  a.D0 = p->d_D0;
  a.kd = p->d_kd;
  a.kf = (const Real*)p->d_kf;
  a.pulse = p->d_pulse;
  a.sm = p->d_sm;
  a.spos = p->d_spos;
  a.B = p->B;
  a.r = (const Real*)r;
  a.ymeas = (const Real*)ymeas;
  a.gout = (Real*)gout;
  a.scale = scale;
  a.s_in = (const Real*)s_in;
  a.s_out = (Real*)s_out;
  a.eta_over_b = eta_over_b;
  a.alpha = alpha;
  a.stat_part = p->d_stat_part;
  const int grid = (p->g.ntiles + ADJ_WARPS - 1) / ADJ_WARPS;
  adj_kernel<Real, PROX><<<grid, ADJ_WARPS * 32, sm, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  p->launches += 1;
  if (PROX) {
    stats_reduce_kernel<<<1, 256, 0, st>>>(p->d_stat_part, p->g.ntiles, stats);
    CUDA_TRY(cudaGetLastError());
    p->launches += 1;
  }
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
  const int tgmax = dtype == NF_C64 ? TG_MAX_F : TG_MAX_D;
  g.ng = (n_tx + tgmax - 1) / tgmax;
  g.Tg = (n_tx + g.ng - 1) / g.ng;
  for (int i = 0; i < 3; ++i) {
    g.corner[i] = corner[i];
    g.sp[i] = spacing[i];
  }
  p->nvox = (int64_t)g.nx * g.ny * g.nzs;
  p->km = KeyMap{g.T, g.R, g.F, g.Tg};
  p->KS = g.ng * g.R * g.Tg * g.F;
  p->ksblocks = (p->KS + 1023) / 1024;
  p->fwd_gridx = (g.ntiles + FWD_WARPS - 1) / FWD_WARPS;
  const size_t rs = real_size(p);
  {
    // bound the forward partial buffer to ~512 MB
    long long ch = (512LL << 20) / ((long long)p->fwd_gridx * 2 * rs);
    ch = std::max<long long>(ch, 1024);
    ch = std::min<long long>(ch, max_batch);
    p->fwd_chunk = (int)ch;
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
#define ALLOC(ptr, bytes)                  \
  if ((rc = dalloc(p, &(ptr), (bytes)))) { \
    free_plan(p);                          \
    return rc;                             \
  }
  ALLOC(p->d_ant, sizeof(double) * 3 * g.A);
  ALLOC(p->d_kd, sizeof(double) * n_f);
  ALLOC(p->d_kf, rs * n_f);
  ALLOC(p->d_pulse, sizeof(double) * 2 * n_f);
  ALLOC(p->d_tab, rs * (size_t)g.ntiles * g.A * 2 * 32 * V);
  ALLOC(p->d_D0, sizeof(double) * (size_t)g.ntiles * g.A);
  ALLOC(p->d_pos_of_key, sizeof(int) * (size_t)p->KS);
  ALLOC(p->d_cnt, sizeof(int) * (size_t)p->ksblocks);
  ALLOC(p->d_sm, sizeof(int) * (size_t)max_batch);
  ALLOC(p->d_spos, sizeof(int) * (size_t)max_batch);
  ALLOC(p->d_partials, 2 * rs * (size_t)p->fwd_gridx * p->fwd_chunk);
  ALLOC(p->d_stat_part, sizeof(double) * 4 * (size_t)std::max(g.ntiles, 1024));
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
  if (cudaMemset(p->d_pos_of_key, 0xff, sizeof(int) * (size_t)p->KS) != cudaSuccess) {
    free_plan(p);
    return fail(NF_ERR_CUDA, "cudaMemset pos_of_key");
  }
  dim3 grid(g.ntiles, g.A);
  if (dtype == NF_C64)
    build_table_kernel<float><<<grid, 32>>>(g, p->d_ant, (float*)p->d_tab, p->d_D0);
  else
    build_table_kernel<double><<<grid, 32>>>(g, p->d_ant, (double*)p->d_tab, p->d_D0);
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
  info[5] = p->fwd_gridx;
  info[6] = p->dtype;
  info[7] = p->launches;
  return NF_OK;
}

int nf_batch_prepare(nf_plan* p, const int32_t* idx, int B, void* stream) {
  if (!p || !idx) return fail(NF_ERR_ARG, "null argument");
  if (B < 1) return fail(NF_ERR_ARG, "channel subset must be non-empty");
  if (B > p->max_batch) return fail(NF_ERR_ARG, "batch larger than the plan's max_batch");
  cudaStream_t st = (cudaStream_t)stream;
  mark_kernel<<<(B + 255) / 256, 256, 0, st>>>(p->km, idx, B, p->d_pos_of_key);
  count_kernel<<<p->ksblocks, 1024, 0, st>>>(p->d_pos_of_key, p->KS, p->d_cnt);
  scan_kernel<<<1, 1024, 0, st>>>(p->d_cnt, p->ksblocks);
  compact_kernel<<<p->ksblocks, 1024, 0, st>>>(p->km, p->d_pos_of_key, p->KS, p->d_cnt, p->d_sm, p->d_spos);
  CUDA_TRY(cudaGetLastError());
  p->launches += 4;
  p->B = B;
  return NF_OK;
}

int nf_forward(nf_plan* p, const void* s, void* y, void* stream) {
  if (!p || !s || !y) return fail(NF_ERR_ARG, "null argument");
  if (p->B < 1) return fail(NF_ERR_STATE, "no batch staged (call nf_batch_prepare first)");
  cudaStream_t st = (cudaStream_t)stream;
  return p->dtype == NF_C64 ? launch_forward<float>(p, s, y, st) : launch_forward<double>(p, s, y, st);
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

int nf_sample_flat(nf_plan* p, uint64_t seed, uint64_t iter, int B, int32_t* idx, void* stream) {
  if (!p || !idx) return fail(NF_ERR_ARG, "null argument");
  if (B < 1 || B > p->M) return fail(NF_ERR_ARG, "batch must be in [1, M]");
  int bits = 2;
  while ((1LL << bits) < p->M) bits += 2;
  const uint64_t key = (seed * 0x9E3779B97F4A7C15ULL) ^ (iter * 0xD1B54A32D192ED03ULL) ^ 0x2545F4914F6CDD1DULL;
  sample_kernel<<<(B + 255) / 256, 256, 0, (cudaStream_t)stream>>>(key, bits / 2, p->M, B, idx);
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
