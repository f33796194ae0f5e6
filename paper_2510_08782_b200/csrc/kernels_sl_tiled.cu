// kernels_sl_tiled.cu — shared-memory z-marching semi-Lagrangian kernels (sm_100a, d = 3).
//
// Same arithmetic as kernels_sl.cu (readings R5-R7): out(l) =
// I[in](l + delta(l)) with the periodic tricubic Lagrange stencil, but the 64 taps are
// gathered from shared memory instead of L1.  A block owns an output tile of 32 (x) x 8 (y)
// columns and marches through a chunk of z planes; the input planes around the current
// plane (tile + halo 4 in x, H in y/z) live in a ring of shared-memory slots.  One thread
// per output point per plane: a warp is one 128-byte x row of outputs, so the delta / E /
// output streams stay fully coalesced; smem rows have a 64-word pitch, so lanes of a warp
// that straddle two rows / planes hit disjoint banks.  Feet whose floor offsets leave the
// halo fall back to the L1 gather for that point (correct for any CFL).
//
// Single-field kernels (SL step, last step, Heun factor): k_sl_pipe, a cp.async pipeline.
//   * the ring has NZR = 2H + 2K = 16 slots (slot = plane & 15); the K planes of stage i+1
//     are copied global -> shared with cp.async (no register staging, no loader role)
//     while stage i is computed;
//   * ONE barrier per stage: after it every thread has finished stage
//     i-1, whose oldest K slots are refilled with stage i+1's planes (prefetch distance one
//     stage of K = 4 planes, NZR >= 2H + 2K) — half the barriers of a wait/refill pair;
//   * the per-point streams (delta, E) are prefetched into registers one plane ahead.
//   * x window: warps whose x floors take two values read 5 columns at lane-uniform offsets
//     (conflict-free) instead of 4 at per-lane offsets (a 33-column span: 2 wavefronts/tap).
// Trace (3 fields, RK2 midpoint feet, H = 2: the midpoint displacement dt/2 v has |floor| <= 1):
// k_sl_trace2 (default) computes column pairs (z, z+1) from a fixed 5 x 5 x 6 window shared by
// both feet and both points; k_sl_trace (TOPT_TRACE2=0) one point per thread per plane.
#include <cmath>

#include "internal.cuh"

namespace topt {

namespace tiled {
constexpr int TX = 32, TY = 8;
constexpr int XH = 4;            // x halo (float4 aligned): foot floors in [-3, 2]
constexpr int XW = TX + 2 * XH;  // 40 floats loaded per row
constexpr int PW = 64;           // smem row pitch: a multiple of 32 words
template <int H>                 // y/z halo: foot floors in [-H+1, H-2]
struct Cfg {
  static constexpr int PH = TY + 2 * H;  // rows per plane
  static constexpr int PS = PW * PH;     // floats per plane (multiple of 32)
};
}  // namespace tiled

enum { M_STEP = 0, M_LAST = 1, M_EFACTOR = 2, M_TRACE = 3 };

struct TileArgs {
  const float* in[3];   // fields gathered with one stencil (TRACE: v components)
  const float* delta;   // 3F displacement in cells (not TRACE)
  const float* E;       // optional factor (STEP / LAST)
  const float* m1;      // LAST
  float* out[2];        // STEP/LAST/EFACTOR: out[0]; TRACE: out[0] = delta_f, out[1] = delta_a (3F each)
  float* lamS;          // LAST (may be null)
  double* partials;     // LAST / TRACE
  float sh, h2;         // EFACTOR: E = 1 + sh (a + b) + h2 a b
};

// Cubic Lagrange weights on nodes -1, 0, 1, 2 (R5) in 8 operations: with a = t (t - 1),
// w0 = a (2 - t)/6, w1 = (t - 1)(a - 2)/2, w2 = -t (a - 2)/2, w3 = a (t + 1)/6.
// t = 0 gives exactly (0, 1, 0, 0) (v = 0 is a bitwise identity).
__device__ __forceinline__ void lag4(float t, float w[4]) {
  const float a = fmaf(t, t, -t);
  const float c6 = a * (1.0f / 6.0f), c3 = a * (1.0f / 3.0f);
  const float h = fmaf(a, 0.5f, -1.0f);
  w[0] = fmaf(-t, c6, c3);
  w[1] = fmaf(t, h, -h);
  w[2] = -t * h;
  w[3] = fmaf(t, c6, c6);
}

// The same weights for two axes at once in packed fp32x2 (8 FFMA2/FMUL2 instead of 16 scalar
// operations; identical IEEE roundings, so bitwise the scalar lag4's).
__device__ __forceinline__ void lag4x2(float2 t, float2 w[4]) {
  const float2 a = __ffma2_rn(t, t, make_float2(-t.x, -t.y));
  const float2 c6 = __fmul2_rn(a, make_float2(1.0f / 6.0f, 1.0f / 6.0f));
  const float2 c3 = __fmul2_rn(a, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
  const float2 h = __ffma2_rn(a, make_float2(0.5f, 0.5f), make_float2(-1.0f, -1.0f));
  const float2 mt = make_float2(-t.x, -t.y);
  w[0] = __ffma2_rn(mt, c6, c3);
  w[1] = __ffma2_rn(t, h, make_float2(-h.x, -h.y));
  w[2] = __fmul2_rn(mt, h);
  w[3] = __ffma2_rn(t, c6, c6);
}
#ifndef TOPT_SL_PACKW
#define TOPT_SL_PACKW 0  // packed x/y (trace: A/B) weights: measured no gain (SL step 1877 -> 1857 GB/s)
#endif
// x, y and z weights of one stencil (x and y packed)
__device__ __forceinline__ void lag4_xyz(float tx, float ty, float tz, float wx[4], float wy[4], float wz[4]) {
#if TOPT_SL_PACKW
  float2 w[4];
  lag4x2(make_float2(tx, ty), w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    wx[k] = w[k].x;
    wy[k] = w[k].y;
  }
#else
  lag4(tx, wx);
  lag4(ty, wy);
#endif
  lag4(tz, wz);
}

// base + idx (idx < 2^32 floats) as ONE mad.wide.u32 (the generic form costs a 32-bit add and
// a 64-bit shift-add pair per address)
template <typename T>
__device__ __forceinline__ T* at_u32(T* base, unsigned idx) {
  T* r;
  asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(r) : "r"(idx), "l"(base));
  return r;
}

// Global-memory (L1) gather, periodic; fallback for feet outside the halo.
__device__ __forceinline__ float gather_global(const Geom& g, const float* __restrict__ f, int x, int y, int z,
                                               float dx, float dy, float dz) {
  const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
  const int ix = x + (int)fx, iy = y + (int)fy;
  int iz = z + (int)fz;
  if (g.zh && (iz - 1 < -g.zh || iz + 2 >= g.nz + g.zh)) {  // foot beyond the slab's halo / window
    if (!g.nzw) {
      if (g.haloerr) *g.haloerr = 1;  // the host sizes the window from max |delta_z|: never reached
      return 0.0f;
    }
    // the window covers a whole period: wrap iz into [-zh + 1, nzw - zh] (periodic in z)
    int r = (iz + g.zh - 1) % g.nzw;
    if (r < 0) r += g.nzw;
    iz = r - g.zh + 1;
    TOPT_DEVICE_CHECK(iz - 1 >= -g.zh && iz + 2 < g.nz + g.zh);
  }
  float wx[4], wy[4], wz[4];
  lag4(dx - fx, wx);
  lag4(dy - fy, wy);
  lag4(dz - fz, wz);
  float acc = 0.0f;
  for (int c = 0; c < 4; ++c) {
    const size_t zb = (size_t)(g.zh ? iz - 1 + c + g.zh : ((iz - 1 + c) & (g.nz - 1))) * g.ny;
    float rc = 0.0f;
    for (int b = 0; b < 4; ++b) {
      const float* row = f + (zb + ((iy - 1 + b) & (g.ny - 1))) * g.nx;
      float s = 0.0f;
      for (int a = 0; a < 4; ++a) s = fmaf(wx[a], __ldg(row + ((ix - 1 + a) & (g.nx - 1))), s);
      rc = fmaf(wy[b], s, rc);
    }
    acc = fmaf(wz[c], rc, acc);
  }
  return acc;
}

#ifndef TOPT_SL_XFIRST
#define TOPT_SL_XFIRST 1  // gather_smem contracts x first (no per-tap x*y weight products; +1% SL step)
#endif
// 64-tap tricubic gather of NF fields from smem planes (field stride FS floats); slot(c) =
// smem offset of plane c (c = 0..3: planes iz-1 .. iz+2), rowoff = offset of the first tap.
// Planes are taken in pairs (c, c+1) by packed fp32x2 FMAs with the x-y weight product
// (one FMUL2 per tap, shared by both pairs): acc_{01} = sum_ab wx_a wy_b (f_{ab,0}, f_{ab,1}),
// then the z weights (4 FMAs).
template <int NF, int FS, typename SlotF>
__device__ __forceinline__ void gather_smem(const float* sm, SlotF slot, int rowoff, const float wx[4],
                                            const float wy[4], const float wz[4], float* res) {
  using tiled::PW;
  float2 wx2[4], wy2[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    wx2[a] = make_float2(wx[a], wx[a]);
    wy2[a] = make_float2(wy[a], wy[a]);
  }
  const int p0 = slot(0) + rowoff, p1 = slot(1) + rowoff, p2 = slot(2) + rowoff, p3 = slot(3) + rowoff;
#if TOPT_SL_XFIRST
  // contraction x, then y, then z: 32 + 8 FFMA2 per field (no per-tap weight products)
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const float* s0 = sm + f * FS;
    float2 lo = make_float2(0.f, 0.f), hi = lo;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int o = b * PW;
      float2 r01 = __fmul2_rn(wx2[0], make_float2(s0[p0 + o], s0[p1 + o]));
      float2 r23 = __fmul2_rn(wx2[0], make_float2(s0[p2 + o], s0[p3 + o]));
#pragma unroll
      for (int a = 1; a < 4; ++a) {
        r01 = __ffma2_rn(wx2[a], make_float2(s0[p0 + o + a], s0[p1 + o + a]), r01);
        r23 = __ffma2_rn(wx2[a], make_float2(s0[p2 + o + a], s0[p3 + o + a]), r23);
      }
      lo = b ? __ffma2_rn(wy2[b], r01, lo) : __fmul2_rn(wy2[b], r01);
      hi = b ? __ffma2_rn(wy2[b], r23, hi) : __fmul2_rn(wy2[b], r23);
    }
    res[f] = fmaf(wz[3], hi.y, fmaf(wz[2], hi.x, fmaf(wz[1], lo.y, wz[0] * lo.x)));
  }
#else
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const float* s0 = sm + f * FS;
    float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int o = b * PW + a;
        const float2 w = __fmul2_rn(wx2[a], wy2[b]);
        lo = (a | b) ? __ffma2_rn(w, make_float2(s0[p0 + o], s0[p1 + o]), lo)
                     : __fmul2_rn(w, make_float2(s0[p0 + o], s0[p1 + o]));
        hi = (a | b) ? __ffma2_rn(w, make_float2(s0[p2 + o], s0[p3 + o]), hi)
                     : __fmul2_rn(w, make_float2(s0[p2 + o], s0[p3 + o]));
      }
    res[f] = fmaf(wz[3], hi.y, fmaf(wz[2], hi.x, fmaf(wz[1], lo.y, wz[0] * lo.x)));
  }
#endif
}

__device__ __forceinline__ void cp_async16(float* smem, const float* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// =====================================================================================
// Single-field pipelined kernel (STEP / LAST / EFACTOR).
// =====================================================================================
#ifndef TOPT_SL_HALO
#define TOPT_SL_HALO 4
#endif
namespace pipe {
#ifndef TOPT_SL_K
#define TOPT_SL_K 4
#endif
#ifndef TOPT_SL_D
#define TOPT_SL_D 1
#endif
constexpr int H = TOPT_SL_HALO, K = TOPT_SL_K;  // y/z halo; planes per pipeline stage
#ifndef TOPT_SL_JUNROLL
#define TOPT_SL_JUNROLL 1
#endif
constexpr int JU = TOPT_SL_JUNROLL;             // unroll of the per-plane loop of a stage
constexpr int D = TOPT_SL_D;                    // prefetch distance in stages (one barrier per stage)
constexpr int NZR = 16;                         // ring slots (power of two)
// the planes of stage st+D are copied at the top of stage st, over planes only stages < st need
static_assert(NZR >= 2 * H + (D + 1) * K, "ring too small");
constexpr int PS = tiled::Cfg<H>::PS, PH = tiled::Cfg<H>::PH;
constexpr int NF4 = PH * (tiled::XW / 4);  // float4 per plane
constexpr size_t SMEM = (size_t)NZR * PS * sizeof(float);
static_assert(H % K == 0, "stages of K planes tile the halo");
}  // namespace pipe

#ifndef TOPT_TRACE2
#define TOPT_TRACE2 1  // z-pair trace kernel (k_sl_trace2)
#endif
#ifndef TOPT_SL_XWIN
#define TOPT_SL_XWIN 1  // warp-uniform 5-column x window when the warp's x floors span two values
#endif
#ifndef TOPT_SL_XWIN_TEST
#define TOPT_SL_XWIN_TEST 1  // ... only when the per-lane path would have bank conflicts
#endif
#ifndef TOPT_SL_XWIN6
#define TOPT_SL_XWIN6 1  // 6-column window for warps whose x floors take three values (+2% SL step)
#endif
// x-window gather of k_sl_pipe: every lane reads the NC columns starting at the warp's common
// offset (row pointer s), its 4 x weights placed at offset sh = ix - min(ix) of an NC-vector
// (zeros elsewhere); planes p0 .. p0+3 (ring slots), contraction x, then y, then z.
template <int NC>
__device__ __forceinline__ float xwin_gather(const float* s, int p0, int sh, const float wx[4], const float wy[4],
                                             const float wz[4]) {
  using pipe::NZR;
  using pipe::PS;
  using tiled::PW;
  float wn[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    float w = 0.0f;
#pragma unroll
    for (int q = 0; q <= NC - 4; ++q)
      if (k - q >= 0 && k - q < 4) w = sh == q ? wx[k - q] : w;
    wn[k] = w;
  }
  const float* s0 = s + ((p0) & (NZR - 1)) * PS;
  const float* s1 = s + ((p0 + 1) & (NZR - 1)) * PS;
  const float* s2 = s + ((p0 + 2) & (NZR - 1)) * PS;
  const float* s3 = s + ((p0 + 3) & (NZR - 1)) * PS;
  float2 lo = make_float2(0.f, 0.f), hi = lo;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float2 r01 = make_float2(0.f, 0.f), r23 = r01;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int oo = b * PW + k;
      const float2 w = make_float2(wn[k], wn[k]);
      r01 = __ffma2_rn(w, make_float2(s0[oo], s1[oo]), r01);
      r23 = __ffma2_rn(w, make_float2(s2[oo], s3[oo]), r23);
    }
    const float2 wb = make_float2(wy[b], wy[b]);
    lo = __ffma2_rn(wb, r01, lo);
    hi = __ffma2_rn(wb, r23, hi);
  }
  return fmaf(wz[3], hi.y, fmaf(wz[2], hi.x, fmaf(wz[1], lo.y, wz[0] * lo.x)));
}

#ifndef TOPT_SL_MINB
#define TOPT_SL_MINB 3  // resident blocks per SM the register budget is sized for
#endif
template <int MODE, bool HAS_E>
__global__ void __launch_bounds__(256, TOPT_SL_MINB) k_sl_pipe(Geom g, int ZC, TileArgs a) {
  using namespace tiled;
  using pipe::H;
  using pipe::K;
  using pipe::NZR;
  using pipe::PS;
  extern __shared__ __align__(16) float sm[];  // [NZR][PH][PW]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tilesx = g.nx / TX, tilesy = g.ny / TY;
  int bid = blockIdx.x;
  const int bx = bid % tilesx;
  bid /= tilesx;
  const int by = bid % tilesy;
  bid /= tilesy;
  const int z0 = bid * ZC;
  const int x0 = bx * TX, y0 = by * TY;
  const size_t F = g.F;
  const size_t plane = (size_t)g.nx * g.ny;
  const float* __restrict__ in = a.in[0];

  auto psrc = [&](int pl) -> size_t { return (size_t)(g.zh ? pl + g.zh : (pl & (g.nz - 1))) * plane; };
  // ring fill by cp.async: a stage is K consecutive planes [pa, pa + K) (pa a multiple of K, so
  // the planes are contiguous in the source, wrapped or halo'd, and land in one aligned slot group).
  // Thread t owns float4 elements t + 256 j of the stage; their plane / row / column offsets are
  // fixed, so per stage only the stage's source base and slot base are computed (32-bit offsets).
  constexpr int NJ = (K * pipe::NF4 + 255) / 256;
  unsigned soff[NJ], goff[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int i = threadIdx.x + 256 * j, jo = i / pipe::NF4, rem = i % pipe::NF4;
    const int r = rem / (XW / 4), k = rem % (XW / 4);
    soff[j] = (unsigned)(jo * PS + r * PW + 4 * k) * 4u;
    goff[j] = (unsigned)jo * (unsigned)plane +
              (unsigned)(((y0 - H + r) & (g.ny - 1)) * g.nx + ((x0 - XH + 4 * k) & (g.nx - 1)));
  }
  const unsigned sm0 = (unsigned)__cvta_generic_to_shared(sm);
  auto load_stage = [&](int pa) {  // planes [pa, pa + K)
    const float* src = in + psrc(pa);
    const unsigned sb = sm0 + (unsigned)((pa & (NZR - 1)) * PS) * 4u;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      if (threadIdx.x + 256 * j < K * pipe::NF4) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb + soff[j]), "l"(src + goff[j]));
  };

  const int nst = ZC / K;
  for (int p = z0 - H; p < z0 + K + H; p += K) load_stage(p);  // stage 0's planes
  cp_commit();
  for (int u = 1; u < pipe::D; ++u) {  // stages 1 .. D-1
    if (u < nst) load_stage(z0 + u * K + H);
    cp_commit();
  }

  const size_t gi0 = (size_t)z0 * plane + (size_t)(y0 + ty) * g.nx + x0 + tx;
  // per-thread stream bases; offsets from them fit 32 bits (3F < 2^32 for every supported grid)
  const float* __restrict__ pd = a.delta + gi0;
  const float* __restrict__ pE = HAS_E ? a.E + gi0 : nullptr;
  float* __restrict__ pout = a.out[0] + gi0;
  const unsigned F32 = (unsigned)F, P32 = (unsigned)plane;
  // per-point streams (delta_x, delta_y, delta_z, E), prefetched one plane ahead
  float n0, n1, n2, nE = 1.0f;
  auto fetch = [&](int zi) {
    const unsigned o = (unsigned)zi * P32;
    n0 = __ldg(at_u32(pd, o));
    n1 = __ldg(at_u32(pd, F32 + o));
    n2 = __ldg(at_u32(pd, 2u * F32 + o));
    if (HAS_E) nE = __ldg(at_u32(pE, o));
  };
  fetch(0);
  double acc = 0.0;

#pragma unroll 1
  for (int st = 0; st < nst; ++st) {
    // one barrier per stage: after it every thread has finished stage st-1, whose oldest
    // K slots (planes needed by no later stage, NZR >= 2H + (D+1)K) take stage st+D's planes
    TOPT_STRESS_POINT(st * 3 + 11);
    cp_wait<pipe::D - 1>();
    __syncthreads();
    if (st + pipe::D < nst) load_stage(z0 + (st + pipe::D) * K + H);
    cp_commit();
    TOPT_STRESS_POINT(st * 3 + 12);
#pragma unroll pipe::JU
    for (int j = 0; j < K; ++j) {
      const int zi = st * K + j, z = z0 + zi;
      const unsigned o = (unsigned)zi * P32;
      const float dx = n0, dy = n1, dz = n2, cE = nE;
      if (zi + 1 < ZC) fetch(zi + 1);
      const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
      const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
      float r;
      // resident ring planes during stage st: [z0 + st K - H, z0 + st K + K + H)
      TOPT_DEVICE_CHECK(!(iz >= -H + 1 && iz <= H - 2) ||
                        (z + iz - 1 >= z0 + st * K - H && z + iz + 2 < z0 + st * K + K + H));
      const bool inr = !(ix < -XH + 1 || ix > XH - 2 || iy < -H + 1 || iy > H - 2 || iz < -H + 1 || iz > H - 2);
#if TOPT_SL_XWIN
      // x-window path (warp-uniform): when the warp's x floors take exactly two values
      // {mn, mn+1}, the 32 lanes' 4-tap x stencils span 33 columns and EVERY tap of the
      // per-lane path costs two smem wavefronts (columns c and c+32 share a bank).  Instead each
      // lane reads the 5 columns mn-1 .. mn+3 relative to its own x — the same offsets in
      // every lane, so each load is one conflict-free wavefront whatever the lanes' rows and
      // planes — with its 4 x weights at offset ix - mn of a 5-vector: 80 wavefronts per
      // point instead of 128.  Contraction order x, then y, then z.
      const int mn = __reduce_min_sync(0xffffffffu, ix), mx = __reduce_max_sync(0xffffffffu, ix);
      bool win = false;
      if (mx == mn + 1 && __all_sync(0xffffffffu, inr)) {
#if TOPT_SL_XWIN_TEST
        // The per-lane 4-tap path is conflict-free when the lanes' columns tx + ix span < 32
        // AND lanes reading the same column read the same row and plane (a broadcast): with two
        // x floors, only neighbouring lanes can share a column.  That holds for ~55% of these
        // warps (floors falling along x, 256^3 config-4 feet); only the rest pay the window's
        // 80 wavefronts (all-path average 78 -> 71 wavefronts per warp-point).
        const int cl = tx + ix;
        const int span = __reduce_max_sync(0xffffffffu, cl) - __reduce_min_sync(0xffffffffu, cl);
        const unsigned pk = (unsigned)(cl & 0xffff) | ((unsigned)(iy & 0xff) << 16) | ((unsigned)(iz & 0xff) << 24);
        const unsigned nb = __shfl_down_sync(0xffffffffu, pk, 1);
        const bool clash = tx < 31 && ((nb ^ pk) & 0xffffu) == 0u && nb != pk;
        win = span >= 32 || __any_sync(0xffffffffu, clash);
#else
        win = true;
#endif
      }
      if (win) {
        float wx[4], wy[4], wz[4];
        lag4_xyz(dx - fx, dy - fy, dz - fz, wx, wy, wz);
        r = xwin_gather<5>(sm + (ty + iy - 1 + H) * PW + tx + mn - 1 + XH, z + iz - 1, ix - mn, wx, wy, wz);
#if TOPT_SL_XWIN6
      } else if (mx == mn + 2 && __all_sync(0xffffffffu, inr) &&
                 __reduce_max_sync(0xffffffffu, tx + ix) - __reduce_min_sync(0xffffffffu, tx + ix) >= 32) {
        // three x floors whose columns wrap the banks: a 6-column window (96 wavefronts, not 128)
        float wx[4], wy[4], wz[4];
        lag4_xyz(dx - fx, dy - fy, dz - fz, wx, wy, wz);
        r = xwin_gather<6>(sm + (ty + iy - 1 + H) * PW + tx + mn - 1 + XH, z + iz - 1, ix - mn, wx, wy, wz);
#endif
      } else
#endif
      if (!inr) {
        r = gather_global(g, in, x0 + tx, y0 + ty, z, dx, dy, dz);
      } else {
        float wx[4], wy[4], wz[4];
        lag4_xyz(dx - fx, dy - fy, dz - fz, wx, wy, wz);
        const int p0 = z + iz - 1;
        gather_smem<1, 0>(sm, [&](int c) { return ((p0 + c) & (NZR - 1)) * PS; },
                          (ty + iy - 1 + H) * PW + tx + ix - 1 + XH, wx, wy, wz, &r);
      }
      if (MODE == M_EFACTOR) {
        const float bv = sm[(z & (NZR - 1)) * PS + (ty + H) * PW + tx + XH];  // divv(l)
        *at_u32(pout, o) = 1.0f + a.sh * (r + bv) + a.h2 * r * bv;
      } else {
        float val = r;
        if (HAS_E) val *= cE;
        *at_u32(pout, o) = val;
        if (MODE == M_LAST) {
          const size_t gi = gi0 + o;
          const float res = __ldg(a.m1 + gi) - val;
          if (a.lamS) a.lamS[gi] = res;
          acc += (double)res * (double)res;
        }
      }
    }
  }
  cp_wait<0>();

  if (MODE == M_LAST) {
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      a.partials[blockIdx.x] = s;
    }
  }
}

// =====================================================================================
// Trace: both RK2 midpoint feet of the 3 velocity components (R6), fused sum of v.
// =====================================================================================
template <int HALO>
__global__ void __launch_bounds__(256, 2) k_sl_trace(Geom g, int ZC, TileArgs a) {
  using namespace tiled;
  constexpr int NF = 3;
  constexpr int PS = Cfg<HALO>::PS, NZR = 2 * HALO + 2, NLOAD = Cfg<HALO>::PH * (XW / 4);
  extern __shared__ __align__(16) float sm[];  // [NF][NZR][PS]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tilesx = g.nx / TX, tilesy = g.ny / TY;
  int bid = blockIdx.x;
  const int bx = bid % tilesx;
  bid /= tilesx;
  const int by = bid % tilesy;
  bid /= tilesy;
  const int z0 = bid * ZC;
  const int x0 = bx * TX, y0 = by * TY;
  const size_t F = g.F;
  const size_t plane = (size_t)g.nx * g.ny;

  // loader role: thread t < NLOAD owns float4 (row ld_r, chunk ld_k) of every plane
  const bool loader = threadIdx.x < NLOAD;
  const int ld_r = threadIdx.x / (XW / 4), ld_k = threadIdx.x % (XW / 4);
  const size_t ld_off = (size_t)((y0 - HALO + ld_r) & (g.ny - 1)) * g.nx + ((x0 - XH + 4 * ld_k) & (g.nx - 1));
  auto pin = [&](int p) -> size_t { return (size_t)(g.zh ? p + g.zh : (p & (g.nz - 1))) * plane; };
  const int ld_s = ld_r * PW + 4 * ld_k;

#pragma unroll 1
  for (int s = 0; s < 2 * HALO + 1; ++s) {
    if (loader) {
      const size_t po = pin(z0 - HALO + s) + ld_off;
#pragma unroll
      for (int f = 0; f < NF; ++f)
        *reinterpret_cast<float4*>(sm + (f * NZR + s) * PS + ld_s) = __ldg(reinterpret_cast<const float4*>(a.in[f] + po));
    }
  }
  __syncthreads();

  double vs0 = 0.0, vs1 = 0.0, vs2 = 0.0;
  int slot0 = 0;  // ring slot of plane z - HALO
  const size_t gi0 = (size_t)z0 * plane + (size_t)(y0 + ty) * g.nx + x0 + tx;
#pragma unroll 1
  for (int zi = 0; zi < ZC; ++zi) {
    const int z = z0 + zi;
    float4 pre[NF];
    const bool pf = loader && (zi + 1 < ZC);
    if (pf) {
      const size_t po = pin(z + HALO + 1) + ld_off;
#pragma unroll
      for (int f = 0; f < NF; ++f) pre[f] = __ldg(reinterpret_cast<const float4*>(a.in[f] + po));
    }
    const size_t gi = gi0 + (size_t)zi * plane;
    const int cidx = ((slot0 + HALO) % NZR) * PS + (ty + HALO) * PW + tx + XH;
    const float u0 = sm[0 * NZR * PS + cidx];
    const float u1 = sm[1 * NZR * PS + cidx];
    const float u2 = sm[2 * NZR * PS + cidx];
    vs0 += u0; vs1 += u1; vs2 += u2;
    const float c0 = u0 * g.cx, c1 = u1 * g.cy, c2 = u2 * g.cz;
    // Union-window path (warp-uniform): when every lane's midpoint displacement is below one
    // cell per axis (|c/2| < 1), both feet's stencils lie in the FIXED window of nodes -2..2
    // around the point.  Each side's 4 Lagrange weights sit at offset floor + 1 (0 or 1) in a
    // 5-vector, the two sides packed as fp32x2 — one 125-tap pass per component serves both
    // feet, every lane reading consecutive words (no bank conflicts): 375 smem loads per point
    // instead of 384 plus the conflicts of irregular stencils.  Contraction order x, y, z.
    if (__all_sync(0xffffffffu, fabsf(c0) < 2.0f && fabsf(c1) < 2.0f && fabsf(c2) < 2.0f)) {
      float2 W[3][5];
      const float cc[3] = {c0, c1, c2};
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const float dF = 0.5f * -1.0f * cc[ax], dA = 0.5f * 1.0f * cc[ax];  // as the per-side path
        const float fF = floorf(dF), fA = floorf(dA);
        float wF[4], wA[4];
        lag4(dF - fF, wF);
        lag4(dA - fA, wA);
        const bool sF = fF == 0.0f, sA = fA == 0.0f;  // offset 1 (floor 0) or 0 (floor -1)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const float f0 = k < 4 ? wF[k] : 0.0f, f1 = k > 0 ? wF[k - 1] : 0.0f;
          const float a0 = k < 4 ? wA[k] : 0.0f, a1 = k > 0 ? wA[k - 1] : 0.0f;
          W[ax][k] = make_float2(sF ? f1 : f0, sA ? a1 : a0);
        }
      }
      const int rbase = (ty - 2 + HALO) * PW + tx - 2 + XH;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        float2 res = make_float2(0.f, 0.f);
#pragma unroll
        for (int cz = 0; cz < 5; ++cz) {
          int sl = slot0 + HALO - 2 + cz;
          if (sl >= NZR) sl -= NZR;
          const float* pp = sm + (f * NZR + sl) * PS + rbase;
          float2 pl = make_float2(0.f, 0.f);
#pragma unroll
          for (int by = 0; by < 5; ++by) {
            float2 row = __fmul2_rn(W[0][0], make_float2(pp[by * PW], pp[by * PW]));
#pragma unroll
            for (int ax = 1; ax < 5; ++ax) {
              const float sv = pp[by * PW + ax];
              row = __ffma2_rn(W[0][ax], make_float2(sv, sv), row);
            }
            pl = __ffma2_rn(W[1][by], row, pl);
          }
          res = __ffma2_rn(W[2][cz], pl, res);
        }
        const float sc = f == 0 ? g.cx : (f == 1 ? g.cy : g.cz);
        if (a.out[0]) a.out[0][f * F + gi] = -1.0f * sc * res.x;
        if (a.out[1]) a.out[1][f * F + gi] = 1.0f * sc * res.y;
      }
    } else
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      float* o = a.out[side];
      if (!o) continue;
      const float sg = side == 0 ? -1.0f : 1.0f;
      const float dx = 0.5f * sg * c0, dy = 0.5f * sg * c1, dz = 0.5f * sg * c2;
      const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
      const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
      float r[NF];
      if (ix < -XH + 1 || ix > XH - 2 || iy < -HALO + 1 || iy > HALO - 2 || iz < -HALO + 1 || iz > HALO - 2) {
#pragma unroll
        for (int f = 0; f < NF; ++f) r[f] = gather_global(g, a.in[f], x0 + tx, y0 + ty, z, dx, dy, dz);
      } else {
        float wx[4], wy[4], wz[4];
        lag4(dx - fx, wx);
        lag4(dy - fy, wy);
        lag4(dz - fz, wz);
        const int s0 = slot0 + HALO + iz - 1;
        gather_smem<NF, NZR * PS>(sm, [&](int c) { int s = s0 + c; if (s >= NZR) s -= NZR; return s * PS; },
                                  (ty + iy - 1 + HALO) * PW + tx + ix - 1 + XH, wx, wy, wz, r);
      }
      o[gi] = sg * g.cx * r[0];
      o[F + gi] = sg * g.cy * r[1];
      o[2 * F + gi] = sg * g.cz * r[2];
    }
    if (pf) {
      int ps = slot0 + 2 * HALO + 1;
      if (ps >= NZR) ps -= NZR;
#pragma unroll
      for (int f = 0; f < NF; ++f) *reinterpret_cast<float4*>(sm + (f * NZR + ps) * PS + ld_s) = pre[f];
    }
    if (++slot0 == NZR) slot0 = 0;
    __syncthreads();
  }

  if (a.partials) {
    __shared__ double redv[3][8];
    double v3[3] = {vs0, vs1, vs2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double t = v3[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
      if ((threadIdx.x & 31) == 0) redv[c][threadIdx.x >> 5] = t;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += redv[threadIdx.x][w];
      a.partials[(size_t)threadIdx.x * kMaxPartials + blockIdx.x] = t;
    }
  }
}

// =====================================================================================
// Trace, z-pair form (k_sl_trace2): a thread computes the feet of the points (z, z+1) of its
// column.  When every lane of the warp has |c/2| < 1 per axis for both points (c = dt v/h in
// cells), the four stencils (2 points x 2 sides) lie in the FIXED window of nodes -2..2 in
// x and y and planes z-2 .. z+3: each window row (5 consecutive words, the same offsets in
// every lane: conflict-free) is loaded ONCE and contracted with both points' x weights
// (forward/adjoint packed as fp32x2) — 150 smem loads per component per pair instead of
// 250.  Otherwise the pair takes the per-point paths of k_sl_trace.  The 8-slot plane ring is
// filled with cp.async, two planes per step, one barrier per pair.
// =====================================================================================
#ifndef TOPT_TRACE_MIRROR
#define TOPT_TRACE_MIRROR 1  // mirrored-operand fast path of k_sl_trace2 (fewer FMAs, see below)
#endif
// Mirrored-operand form of a point's two midpoint stencils (k_sl_trace2 fast path).  On the
// window nodes 0..4 (offsets -2..2) the adjoint weights a5 have support {1,2,3,e} (e = 4 when
// the adjoint floor is 0, else 0) and the forward weights are a5 reversed (w_k(1-t) = w_{3-k}(t)).
// So forward = sum_k a5[k] f[4-k] and adjoint = sum_k a5[k] f[k]: ONE scalar weight times the
// operand pair (f[4-k], f[k]) gives both sides, with 4 terms per axis instead of the union
// window's 5 packed ones.  x and y use this (the pair's two rows / columns are loaded per lane);
// z keeps the packed (forward, adjoint) weights over the 5 window planes.
struct MirrorW {
  float ax[3], axe;  // a5_x[1..3], a5_x[e_x]
  float ay[3], aye;  // a5_y[1..3], a5_y[e_y]
  float2 wz[5];      // (a5_z[4-c], a5_z[c])
};
// axis `ax` of a point's MirrorW from its adjoint floor fA and lag4 weights w
__device__ __forceinline__ void mirror_axis(float fA, const float w[4], int ax, MirrorW& m) {
  const bool sA = fA == 0.0f;
  if (ax < 2) {
    float* a = ax == 0 ? m.ax : m.ay;
#pragma unroll
    for (int k = 0; k < 3; ++k) a[k] = sA ? w[k] : w[k + 1];
    (ax == 0 ? m.axe : m.aye) = sA ? w[3] : w[0];
  } else {
    float a5[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) a5[k] = sA ? (k > 0 ? w[k - 1] : 0.0f) : (k < 4 ? w[k] : 0.0f);
#pragma unroll
    for (int k = 0; k < 5; ++k) m.wz[k] = make_float2(a5[4 - k], a5[k]);
  }
}
// both points of a pair: the weights of A and B per axis in one packed lag4x2
__device__ __forceinline__ void mirror_weights2(const float ccA[3], const float ccB[3], MirrorW& mA, MirrorW& mB) {
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const float dA = 0.5f * ccA[ax], dB = 0.5f * ccB[ax];
    const float fA = floorf(dA), fB = floorf(dB);
    float wA[4], wB[4];
#if TOPT_SL_PACKW
    float2 w[4];
    lag4x2(make_float2(dA - fA, dB - fB), w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      wA[k] = w[k].x;
      wB[k] = w[k].y;
    }
#else
    lag4(dA - fA, wA);
    lag4(dB - fB, wB);
#endif
    mirror_axis(fA, wA, ax, mA);
    mirror_axis(fB, wB, ax, mB);
  }
}
#ifndef TOPT_TRACE_MINB
#define TOPT_TRACE_MINB 2
#endif
__global__ void __launch_bounds__(256, TOPT_TRACE_MINB) k_sl_trace2(Geom g, int ZC, TileArgs a) {
  using namespace tiled;
  constexpr int HALO = 2, NF = 3, NZR = 8;
  constexpr int PS = Cfg<HALO>::PS, PH = Cfg<HALO>::PH, NF4 = PH * (XW / 4);
  extern __shared__ __align__(16) float sm[];  // [NF][NZR][PS]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tilesx = g.nx / TX, tilesy = g.ny / TY;
  int bid = blockIdx.x;
  const int bx = bid % tilesx;
  bid /= tilesx;
  const int by = bid % tilesy;
  bid /= tilesy;
  const int z0 = bid * ZC;
  const int x0 = bx * TX, y0 = by * TY;
  const size_t F = g.F;
  const size_t plane = (size_t)g.nx * g.ny;
  auto psrc = [&](int pl) -> size_t { return (size_t)(g.zh ? pl + g.zh : (pl & (g.nz - 1))) * plane; };
  auto load_planes = [&](int pa, int pb) {  // planes [pa, pb) of the 3 components
    const int n = (pb - pa) * NF * NF4;
    for (int i = threadIdx.x; i < n; i += 256) {
      const int pl = pa + i / (NF * NF4), rem = i % (NF * NF4), f = rem / NF4, q = rem % NF4;
      const int r = q / (XW / 4), k = q % (XW / 4);
      const size_t src = psrc(pl) + (size_t)((y0 - HALO + r) & (g.ny - 1)) * g.nx + ((x0 - XH + 4 * k) & (g.nx - 1));
      cp_async16(sm + (f * NZR + (pl & (NZR - 1))) * PS + r * PW + 4 * k, a.in[f] + src);
    }
  };
  load_planes(z0 - HALO, z0 + 2 + HALO);  // planes of the first pair
  cp_commit();

  double vs0 = 0.0, vs1 = 0.0, vs2 = 0.0;
  const size_t gi0 = (size_t)z0 * plane + (size_t)(y0 + ty) * g.nx + x0 + tx;
  const int rbase = (ty - 2 + HALO) * PW + tx - 2 + XH;
  // (forward, adjoint) weights of one point on window nodes -2..2 per axis.  The two feet of a
  // point are displaced by -c/2 and +c/2 (|c/2| < 1): their fractional offsets are t and 1 - t and
  // their stencils mirror images in the 5-node window, so the forward weights are the adjoint
  // 5-vector reversed (w_k(1 - t) = w_{3-k}(t) for the Lagrange basis on -1..2): one lag4 per axis
  auto weights = [&](const float cc[3], float2 (&W)[3][5]) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const float dA = 0.5f * cc[ax];
      const float fA = floorf(dA);
      float wA[4];
      lag4(dA - fA, wA);
      const bool sA = fA == 0.0f;  // adjoint stencil at window offsets 1..4 (else 0..3)
      float a5[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) a5[k] = sA ? (k > 0 ? wA[k - 1] : 0.0f) : (k < 4 ? wA[k] : 0.0f);
#pragma unroll
      for (int k = 0; k < 5; ++k) W[ax][k] = make_float2(a5[4 - k], a5[k]);
    }
  };
  // per-point, per-side path (k_sl_trace's): stencil at the foot's own floors
  auto single = [&](int z, size_t gi, const float cc[3]) {
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      float* o = a.out[side];
      if (!o) continue;
      const float sg = side == 0 ? -1.0f : 1.0f;
      const float dx = 0.5f * sg * cc[0], dy = 0.5f * sg * cc[1], dz = 0.5f * sg * cc[2];
      const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
      const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
      float r[NF];
      if (ix < -XH + 1 || ix > XH - 2 || iy < -HALO + 1 || iy > HALO - 2 || iz < -HALO + 1 || iz > HALO - 2) {
#pragma unroll
        for (int f = 0; f < NF; ++f) r[f] = gather_global(g, a.in[f], x0 + tx, y0 + ty, z, dx, dy, dz);
      } else {
        float wx[4], wy[4], wz[4];
        lag4(dx - fx, wx);
        lag4(dy - fy, wy);
        lag4(dz - fz, wz);
        const int p0 = z + iz - 1;
        gather_smem<NF, NZR * PS>(sm, [&](int c) { return ((p0 + c) & (NZR - 1)) * PS; },
                                  (ty + iy - 1 + HALO) * PW + tx + ix - 1 + XH, wx, wy, wz, r);
      }
      o[gi] = sg * g.cx * r[0];
      o[F + gi] = sg * g.cy * r[1];
      o[2 * F + gi] = sg * g.cz * r[2];
    }
  };

#pragma unroll 1
  for (int zi = 0; zi < ZC; zi += 2) {
    const int z = z0 + zi;
    TOPT_STRESS_POINT(zi + 21);
    cp_wait<0>();
    __syncthreads();  // planes z-2 .. z+3 resident; everyone is done with the previous pair
    if (zi + 2 < ZC) load_planes(z + 2 + HALO, z + 4 + HALO);  // over planes z-4, z-3
    cp_commit();
    const size_t gA = gi0 + (size_t)zi * plane, gB = gA + plane;
    const int cA = (z & (NZR - 1)) * PS + (ty + HALO) * PW + tx + XH;
    const int cB = ((z + 1) & (NZR - 1)) * PS + (ty + HALO) * PW + tx + XH;
    float ccA[3], ccB[3];
    const float gc[3] = {g.cx, g.cy, g.cz};
    bool ok = true;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const float uA = sm[f * NZR * PS + cA], uB = sm[f * NZR * PS + cB];
      ccA[f] = uA * gc[f];
      ccB[f] = uB * gc[f];
      ok = ok && fabsf(ccA[f]) < 2.0f && fabsf(ccB[f]) < 2.0f;
      if (f == 0) vs0 += (double)uA + (double)uB;
      if (f == 1) vs1 += (double)uA + (double)uB;
      if (f == 2) vs2 += (double)uA + (double)uB;
    }
#if TOPT_TRACE_MIRROR
    // the pair's x and y adjoint floors agree lane by lane (then both points read the same
    // per-lane extra columns / rows): the mirrored-operand path
    const bool sxA = floorf(0.5f * ccA[0]) == 0.0f, syA = floorf(0.5f * ccA[1]) == 0.0f;
    const bool same = sxA == (floorf(0.5f * ccB[0]) == 0.0f) && syA == (floorf(0.5f * ccB[1]) == 0.0f);
    if (__all_sync(0xffffffffu, ok && same)) {
      MirrorW mA, mB;
      mirror_weights2(ccA, ccB, mA, mB);
      // per-lane window offsets: extra column e_x / mirrored 4 - e_x, extra row e_y / 4 - e_y
      const int cE = sxA ? 4 : 0, cM = 4 - cE;
      const int rE = (syA ? 4 : 0) * PW, rM = 4 * PW - rE;
#pragma unroll 1
      for (int f = 0; f < NF; ++f) {
        float2 resA = make_float2(0.f, 0.f), resB = resA;
#pragma unroll
        for (int cz = 0; cz < 6; ++cz) {  // window planes z-2 .. z+3
          const float* pp = sm + (f * NZR + ((z - 2 + cz) & (NZR - 1))) * PS + rbase;
          float r1[3], r2[3], r3[3], re[3], rm[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            r1[k] = pp[PW + 1 + k];
            r2[k] = pp[2 * PW + 1 + k];
            r3[k] = pp[3 * PW + 1 + k];
            re[k] = pp[rE + 1 + k];
            rm[k] = pp[rM + 1 + k];
          }
          const float r1e = pp[PW + cE], r1m = pp[PW + cM], r2e = pp[2 * PW + cE], r2m = pp[2 * PW + cM];
          const float r3e = pp[3 * PW + cE], r3m = pp[3 * PW + cM], ree = pp[rE + cE], rmm = pp[rM + cM];
          // Z_b = sum_k a5_x[k] (f[4-b][4-k], f[b][k]) for b = 1, 3, 2, e_y; plane = sum_b a5_y[b] Z_b
          auto planev = [&](const MirrorW& m) -> float2 {
            const float2 w1 = make_float2(m.ax[0], m.ax[0]), w2 = make_float2(m.ax[1], m.ax[1]);
            const float2 w3 = make_float2(m.ax[2], m.ax[2]), we = make_float2(m.axe, m.axe);
            float2 z1 = __fmul2_rn(w1, make_float2(r3[2], r1[0]));
            z1 = __ffma2_rn(w2, make_float2(r3[1], r1[1]), z1);
            z1 = __ffma2_rn(w3, make_float2(r3[0], r1[2]), z1);
            z1 = __ffma2_rn(we, make_float2(r3m, r1e), z1);
            float2 z3 = __fmul2_rn(w1, make_float2(r1[2], r3[0]));
            z3 = __ffma2_rn(w2, make_float2(r1[1], r3[1]), z3);
            z3 = __ffma2_rn(w3, make_float2(r1[0], r3[2]), z3);
            z3 = __ffma2_rn(we, make_float2(r1m, r3e), z3);
            float2 z2 = __fmul2_rn(w1, make_float2(r2[2], r2[0]));
            z2 = __ffma2_rn(w2, make_float2(r2[1], r2[1]), z2);
            z2 = __ffma2_rn(w3, make_float2(r2[0], r2[2]), z2);
            z2 = __ffma2_rn(we, make_float2(r2m, r2e), z2);
            float2 ze = __fmul2_rn(w1, make_float2(rm[2], re[0]));
            ze = __ffma2_rn(w2, make_float2(rm[1], re[1]), ze);
            ze = __ffma2_rn(w3, make_float2(rm[0], re[2]), ze);
            ze = __ffma2_rn(we, make_float2(rmm, ree), ze);
            float2 y = __fmul2_rn(make_float2(m.ay[0], m.ay[0]), z1);
            y = __ffma2_rn(make_float2(m.ay[1], m.ay[1]), z2, y);
            y = __ffma2_rn(make_float2(m.ay[2], m.ay[2]), z3, y);
            return __ffma2_rn(make_float2(m.aye, m.aye), ze, y);
          };
          if (cz < 5) resA = __ffma2_rn(mA.wz[cz], planev(mA), resA);
          if (cz > 0) resB = __ffma2_rn(mB.wz[cz - 1], planev(mB), resB);
        }
        const float sc = f == 0 ? g.cx : (f == 1 ? g.cy : g.cz);
        if (a.out[0]) {
          a.out[0][f * F + gA] = -1.0f * sc * resA.x;
          a.out[0][f * F + gB] = -1.0f * sc * resB.x;
        }
        if (a.out[1]) {
          a.out[1][f * F + gA] = 1.0f * sc * resA.y;
          a.out[1][f * F + gB] = 1.0f * sc * resB.y;
        }
      }
    } else
#endif
    if (__all_sync(0xffffffffu, ok)) {
      float2 WA[3][5], WB[3][5];
      weights(ccA, WA);
      weights(ccB, WB);
#pragma unroll 1
      for (int f = 0; f < NF; ++f) {
        float2 resA = make_float2(0.f, 0.f), resB = resA;
#pragma unroll
        for (int cz = 0; cz < 6; ++cz) {  // window planes z-2 .. z+3
          const float* pp = sm + (f * NZR + ((z - 2 + cz) & (NZR - 1))) * PS + rbase;
          float2 plA = make_float2(0.f, 0.f), plB = plA;
#pragma unroll
          for (int yb = 0; yb < 5; ++yb) {
            float sv[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) sv[k] = pp[yb * PW + k];
            if (cz < 5) {
              float2 row = __fmul2_rn(WA[0][0], make_float2(sv[0], sv[0]));
#pragma unroll
              for (int k = 1; k < 5; ++k) row = __ffma2_rn(WA[0][k], make_float2(sv[k], sv[k]), row);
              plA = __ffma2_rn(WA[1][yb], row, plA);
            }
            if (cz > 0) {
              float2 row = __fmul2_rn(WB[0][0], make_float2(sv[0], sv[0]));
#pragma unroll
              for (int k = 1; k < 5; ++k) row = __ffma2_rn(WB[0][k], make_float2(sv[k], sv[k]), row);
              plB = __ffma2_rn(WB[1][yb], row, plB);
            }
          }
          if (cz < 5) resA = __ffma2_rn(WA[2][cz], plA, resA);
          if (cz > 0) resB = __ffma2_rn(WB[2][cz - 1], plB, resB);
        }
        const float sc = f == 0 ? g.cx : (f == 1 ? g.cy : g.cz);
        if (a.out[0]) {
          a.out[0][f * F + gA] = -1.0f * sc * resA.x;
          a.out[0][f * F + gB] = -1.0f * sc * resB.x;
        }
        if (a.out[1]) {
          a.out[1][f * F + gA] = 1.0f * sc * resA.y;
          a.out[1][f * F + gB] = 1.0f * sc * resB.y;
        }
      }
    } else {
      single(z, gA, ccA);
      single(z + 1, gB, ccB);
    }
  }
  cp_wait<0>();

  if (a.partials) {
    __shared__ double redv[3][8];
    double v3[3] = {vs0, vs1, vs2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double t = v3[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
      if ((threadIdx.x & 31) == 0) redv[c][threadIdx.x >> 5] = t;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += redv[threadIdx.x][w];
      a.partials[(size_t)threadIdx.x * kMaxPartials + blockIdx.x] = t;
    }
  }
}

// ---- host side ------------------------------------------------------------------------
bool tiled_ok(const Geom& g) {
  return g.d == 3 && g.nx >= tiled::TX && g.nx % tiled::TX == 0 && g.ny % tiled::TY == 0 &&
         g.nz % pipe::K == 0 && (g.zh ? g.nz >= pipe::K : g.nz >= 8);
}

static int num_sms_sl() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// z chunk per block (a multiple of `mult` dividing nz): balance the wave quantisation of
// (tiles x chunks) blocks over the resident slots against the 2H-plane halo re-load.  A halo
// plane is only copied, not computed: weighted 1/4 of a computed plane (fitted to the measured
// 256^3 chunk sizes 8/16/32/64; at 128^3 it moves the SL step from 32- to 8-plane chunks, +5%).
static int tiled_zc(const Geom& g, int H, int mult, int resident) {
  int best = 0;
  double bestc = 1e30;
  for (int zc = 64; zc >= mult; zc >>= 1) {
    if (zc > g.nz || g.nz % zc || zc % mult) continue;
    const double blocks = (double)(g.nx / tiled::TX) * (g.ny / tiled::TY) * (g.nz / zc);
    const double waves = blocks / resident, eff = waves / std::ceil(waves);
    const double cost = (zc + 0.25 * 2.0 * H) / zc / eff;
    if (cost < bestc) { bestc = cost; best = zc; }
  }
  return best ? best : mult;
}

template <typename Kern>
static int resident_blocks(Kern k, int threads, size_t smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
  return (per_sm < 1 ? 1 : per_sm) * num_sms_sl();
}

template <int MODE, bool HAS_E>
static int launch_pipe(const Geom& g, const TileArgs& a, cudaStream_t st) {
  auto kern = k_sl_pipe<MODE, HAS_E>;
  static int resident = 0;
  if (!resident) resident = resident_blocks(kern, 256, pipe::SMEM);
  const int zc = tiled_zc(g, pipe::H, pipe::K, resident);
  const int blocks = (g.nx / tiled::TX) * (g.ny / tiled::TY) * (g.nz / zc);
  kern<<<blocks, 256, pipe::SMEM, st>>>(g, zc, a);
  count_launch();
  return blocks;
}

void tiled_trace(const Geom& g, const float* v, float* df, float* da, double* vsum, int* nparts, cudaStream_t st) {
  constexpr int HALO = 2;  // midpoint displacement dt/2 v: |floor| <= 1 (else L1 fallback)
  TileArgs a{};
  a.partials = vsum;
  // component stride of v: F, or F plus 2 zh halo planes for a halo'd slab copy
  const size_t cs = g.F + 2 * (size_t)g.zh * g.nx * g.ny;
  for (int c = 0; c < 3; ++c) a.in[c] = v + c * cs;
  a.out[0] = df;
  a.out[1] = da;
#if TOPT_TRACE2
  const size_t sm = (size_t)3 * 8 * tiled::Cfg<HALO>::PS * sizeof(float);
  static int resident = 0;
  if (!resident) resident = resident_blocks(k_sl_trace2, 256, sm);
  const int zc = tiled_zc(g, HALO, 2, resident);
  const int blocks = (g.nx / tiled::TX) * (g.ny / tiled::TY) * (g.nz / zc);
  k_sl_trace2<<<blocks, 256, sm, st>>>(g, zc, a);
#else
  const size_t sm = (size_t)3 * (2 * HALO + 2) * tiled::Cfg<HALO>::PS * sizeof(float);
  static int resident = 0;
  if (!resident) resident = resident_blocks(k_sl_trace<HALO>, 256, sm);
  const int zc = tiled_zc(g, HALO, 1, resident);
  const int blocks = (g.nx / tiled::TX) * (g.ny / tiled::TY) * (g.nz / zc);
  k_sl_trace<HALO><<<blocks, 256, sm, st>>>(g, zc, a);
#endif
  count_launch();
  if (nparts) *nparts = blocks;
}

void tiled_step(const Geom& g, const float* in, const float* delta, const float* E, float* out, cudaStream_t st) {
  TileArgs a{};
  a.in[0] = in;
  a.delta = delta;
  a.E = E;
  a.out[0] = out;
  if (E) launch_pipe<M_STEP, true>(g, a, st);
  else launch_pipe<M_STEP, false>(g, a, st);
}

void tiled_last(const Geom& g, const float* in, const float* delta, const float* E, const float* m1, float* mS,
                float* lamS, double* partials, int* nparts, cudaStream_t st) {
  TileArgs a{};
  a.in[0] = in;
  a.delta = delta;
  a.E = E;
  a.m1 = m1;
  a.out[0] = mS;
  a.lamS = lamS;
  a.partials = partials;
  *nparts = E ? launch_pipe<M_LAST, true>(g, a, st) : launch_pipe<M_LAST, false>(g, a, st);
}

void tiled_efactor(const Geom& g, const float* divv, const float* delta, float sh, float h2, float* E,
                   cudaStream_t st) {
  TileArgs a{};
  a.in[0] = divv;
  a.delta = delta;
  a.out[0] = E;
  a.sh = sh;
  a.h2 = h2;
  launch_pipe<M_EFACTOR, false>(g, a, st);
}

}  // namespace topt
