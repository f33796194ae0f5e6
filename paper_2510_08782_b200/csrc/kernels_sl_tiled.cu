// kernels_sl_tiled.cu — shared-memory z-marching semi-Lagrangian kernels (sm_100a, d = 3).
//
// Same arithmetic as kernels_sl.cu (readings R5-R7): out(l) =
// I[in](l + delta(l)) with the periodic tricubic Lagrange stencil, but the 64 taps are
// gathered from shared memory instead of L1:
//   * a block owns an output tile of 32 (x) x 8 (y) columns and marches through ZC planes
//     in z; the input planes z-4 .. z+4 (tile + halo 4 in x and y) live in a ring of 10
//     shared-memory slots; plane z+5 is prefetched into registers while plane z is
//     computed (one float4 per loader thread, coalesced, periodic wrap in x/y/z);
//   * one thread per output point per plane: a warp is one 128-byte x row of outputs, so the
//     delta / E / output streams stay fully coalesced;
//   * feet whose floor offsets leave [-3, 2] in any axis (|delta| > ~3 cells) fall back to
//     the L1 gather of kernels_sl.cu for that point (correct for any CFL).
// Smem rows are padded to a 64-word pitch (bank-conflict-free when a warp straddles rows or
// planes).  Global traffic per output point ~ 1.6 input floats (halo) + the streams.
#include "internal.cuh"

namespace topt {

namespace tiled {
constexpr int TX = 32, TY = 8;
constexpr int XH = 4;                 // x halo (float4 aligned): foot floors in [-3, 2]
constexpr int XW = TX + 2 * XH;       // 40 floats loaded per row
constexpr int PW = 64;                // smem row pitch: a multiple of 32 words, so lanes of a warp that
                                      // straddle two rows / planes hit disjoint banks
template <int H>                      // y/z halo: foot floors in [-H+1, H-2]
struct Cfg {
  static constexpr int PH = TY + 2 * H;       // rows per plane
  static constexpr int PS = PW * PH;          // floats per plane (multiple of 32)
  static constexpr int NZR = 2 * H + 2;       // ring slots (planes z-H .. z+H + one prefetch)
  static constexpr int NLOAD = (XW / 4) * PH; // float4 loads per plane
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
  double* partials;     // LAST
  float sh, h2;         // EFACTOR: E = 1 + sh (a + b) + h2 a b
};

__device__ __forceinline__ void lag4(float t, float w[4]) {
  const float tm1 = t - 1.0f, tm2 = t - 2.0f, tp1 = t + 1.0f;
  w[0] = -t * tm1 * tm2 * (1.0f / 6.0f);
  w[1] = tp1 * tm1 * tm2 * 0.5f;
  w[2] = -tp1 * t * tm2 * 0.5f;
  w[3] = tp1 * t * tm1 * (1.0f / 6.0f);
}

// Global-memory (L1) gather, periodic; fallback for feet outside the halo.
__device__ __forceinline__ float gather_global(const Geom& g, const float* __restrict__ f, int x, int y, int z,
                                               float dx, float dy, float dz) {
  const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
  const int ix = x + (int)fx, iy = y + (int)fy, iz = z + (int)fz;
  if (g.zh && (iz - 1 < -g.zh || iz + 2 >= g.nz + g.zh)) {  // foot beyond the neighbour's halo
    if (g.haloerr) *g.haloerr = 1;
    return 0.0f;
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

template <int MODE, int NF, bool HAS_E, int HALO>
__global__ void __launch_bounds__(256) k_sl_tiled(Geom g, int ZC, TileArgs a) {
  using namespace tiled;
  constexpr int PS = Cfg<HALO>::PS, NZR = Cfg<HALO>::NZR, NLOAD = Cfg<HALO>::NLOAD;
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
  // input plane p (slab-local, may be negative / past nz): periodic wrap, or the halo'd slab buffer
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

  double acc = 0.0, vs0 = 0.0, vs1 = 0.0, vs2 = 0.0;
  int slot0 = 0;  // ring slot of plane z - HALO
  // per-point streams of the current plane, prefetched one plane ahead (hides HBM latency)
  const size_t gi0 = (size_t)z0 * plane + (size_t)(y0 + ty) * g.nx + x0 + tx;
  float nd0 = 0.f, nd1 = 0.f, nd2 = 0.f, nE = 1.f;
  if (MODE != M_TRACE) {
    nd0 = __ldg(a.delta + gi0); nd1 = __ldg(a.delta + F + gi0); nd2 = __ldg(a.delta + 2 * F + gi0);
    if (HAS_E) nE = __ldg(a.E + gi0);
  }
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
    const int x = x0 + tx, y = y0 + ty;
    const size_t gi = gi0 + (size_t)zi * plane;
    const float cd0 = nd0, cd1 = nd1, cd2 = nd2, cE = nE;
    if (MODE != M_TRACE && zi + 1 < ZC) {
      const size_t gn = gi + plane;
      nd0 = __ldg(a.delta + gn); nd1 = __ldg(a.delta + F + gn); nd2 = __ldg(a.delta + 2 * F + gn);
      if (HAS_E) nE = __ldg(a.E + gn);
    }

    // gather NF fields at l + (dx, dy, dz) from the smem ring (or global fallback)
    auto gather = [&](float dx, float dy, float dz, float* res) {
      const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
      const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
      if (ix < -XH + 1 || ix > XH - 2 || iy < -HALO + 1 || iy > HALO - 2 || iz < -HALO + 1 || iz > HALO - 2) {
#pragma unroll
        for (int f = 0; f < NF; ++f) res[f] = gather_global(g, a.in[f], x, y, z, dx, dy, dz);
        return;
      }
      float wx[4], wy[4], wz[4];
      lag4(dx - fx, wx);
      lag4(dy - fy, wy);
      lag4(dz - fz, wz);
      const int rowoff = (ty + iy - 1 + HALO) * PW + tx + ix - 1 + XH;
      int s = slot0 + HALO + iz - 1;
      if (s >= NZR) s -= NZR;
#pragma unroll
      for (int f = 0; f < NF; ++f) res[f] = 0.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int pbase = s * PS + rowoff;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const float* pl = sm + f * NZR * PS + pbase;
          float rc = 0.0f;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const float* r = pl + b * PW;
            float t = wx[0] * r[0];
            t = fmaf(wx[1], r[1], t);
            t = fmaf(wx[2], r[2], t);
            t = fmaf(wx[3], r[3], t);
            rc = fmaf(wy[b], t, rc);
          }
          res[f] = fmaf(wz[c], rc, res[f]);
        }
        if (++s == NZR) s = 0;
      }
    };

    if (MODE == M_TRACE) {
      const int cidx = ((slot0 + HALO) % NZR) * PS + (ty + HALO) * PW + tx + XH;
      const float u0 = sm[0 * NZR * PS + cidx];
      const float u1 = sm[1 * NZR * PS + cidx];
      const float u2 = sm[2 * NZR * PS + cidx];
      vs0 += u0; vs1 += u1; vs2 += u2;
      const float c0 = u0 * g.cx, c1 = u1 * g.cy, c2 = u2 * g.cz;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        float* o = a.out[side];
        if (!o) continue;
        const float sg = side == 0 ? -1.0f : 1.0f;
        float r[NF];
        gather(0.5f * sg * c0, 0.5f * sg * c1, 0.5f * sg * c2, r);
        o[gi] = sg * g.cx * r[0];
        o[F + gi] = sg * g.cy * r[1];
        o[2 * F + gi] = sg * g.cz * r[2];
      }
    } else {
      float r[NF];
      gather(cd0, cd1, cd2, r);
      if (MODE == M_EFACTOR) {
        const float bv = sm[((slot0 + HALO) % NZR) * PS + (ty + HALO) * PW + tx + XH];  // divv(l)
        a.out[0][gi] = 1.0f + a.sh * (r[0] + bv) + a.h2 * r[0] * bv;
      } else {
        float val = r[0];
        if (HAS_E) val *= cE;
        a.out[0][gi] = val;
        if (MODE == M_LAST) {
          const float res = a.m1[gi] - val;
          if (a.lamS) a.lamS[gi] = res;
          acc += (double)res * (double)res;
        }
      }
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

  if (MODE == M_TRACE && a.partials) {
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

bool tiled_ok(const Geom& g) {
  return g.d == 3 && g.nx >= tiled::TX && g.nx % tiled::TX == 0 && g.ny % tiled::TY == 0 &&
         (g.zh ? g.nz >= 1 : g.nz >= 8);
}

static int tiled_zc(const Geom& g) {
  int zc = g.nz < 64 ? g.nz : 64;
  while (g.nz % zc) zc >>= 1;
  return zc;
}

int tiled_blocks(const Geom& g) { return (g.nx / tiled::TX) * (g.ny / tiled::TY) * (g.nz / tiled_zc(g)); }

template <int MODE, int NF, bool HAS_E, int HALO = 4>
static void launch_tiled(const Geom& g, const TileArgs& a, cudaStream_t st) {
  using C = tiled::Cfg<HALO>;
  const size_t sm = (size_t)NF * C::NZR * C::PS * sizeof(float);
  cudaFuncSetAttribute(k_sl_tiled<MODE, NF, HAS_E, HALO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_sl_tiled<MODE, NF, HAS_E, HALO><<<tiled_blocks(g), 256, sm, st>>>(g, tiled_zc(g), a);
  count_launch();
}

void tiled_trace(const Geom& g, const float* v, float* df, float* da, double* vsum, int* nparts, cudaStream_t st) {
  TileArgs a{};
  a.partials = vsum;
  if (nparts) *nparts = tiled_blocks(g);
  // component stride of v: F, or F plus 2 zh halo planes for a halo'd slab copy
  const size_t cs = g.F + 2 * (size_t)g.zh * g.nx * g.ny;
  for (int c = 0; c < 3; ++c) a.in[c] = v + c * cs;
  a.out[0] = df;
  a.out[1] = da;
  launch_tiled<M_TRACE, 3, false, 2>(g, a, st);  // midpoint displacement dt/2 v: |floor| <= 1
}

void tiled_step(const Geom& g, const float* in, const float* delta, const float* E, float* out, cudaStream_t st) {
  TileArgs a{};
  a.in[0] = in;
  a.delta = delta;
  a.E = E;
  a.out[0] = out;
  if (E) launch_tiled<M_STEP, 1, true>(g, a, st);
  else launch_tiled<M_STEP, 1, false>(g, a, st);
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
  *nparts = tiled_blocks(g);
  if (E) launch_tiled<M_LAST, 1, true>(g, a, st);
  else launch_tiled<M_LAST, 1, false>(g, a, st);
}

void tiled_efactor(const Geom& g, const float* divv, const float* delta, float sh, float h2, float* E,
                   cudaStream_t st) {
  TileArgs a{};
  a.in[0] = divv;
  a.delta = delta;
  a.out[0] = E;
  a.sh = sh;
  a.h2 = h2;
  launch_tiled<M_EFACTOR, 1, false>(g, a, st);
}

}  // namespace topt
