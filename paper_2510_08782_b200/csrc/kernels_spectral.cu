// kernels_spectral.cu — pseudo-spectral derivative / body-force kernels and the fused
// 3D-FFT preconditioner (sm_100a), built on the register-resident line FFT of rfft.cuh.
//
// Fourier pseudo-spectral discretisation, operators applied "at
// the cost of two FFTs and a diagonal scaling"; zero spectral entries of L set to 1
// before inversion.  (2.2) P:105-108 body force int lam grad m dt (trapezoid);
// (2.6) P:172 s = -(alpha L)^{-1} g; incompressible Leray projection (R9).
// Readings: R2 (k range), R3 (Nyquist zeroed for odd derivatives / Leray, true value
// in L), R4 (L = |k|^{2p}), R8 (continuity body force), R23 (reg by Parseval).
//
// Every kernel keeps its lines in registers: a thread loads natural positions t + T e of
// its line(s) straight from HBM, transforms, applies the spectral operator at the same
// positions, transforms back and writes / accumulates at the same positions.  Spectra
// between passes are stored in natural order.  Kernels are persistent (grid = resident
// blocks, capped by the work) so the per-thread twiddles are loaded once.
//
// Layout of the complex chain buffers Z_f (F complex each, [n3][n2][n1] like the fields):
//   v-chain (fp64):  (v_x + i v_y) [, (v_z)]      -> (u_x + i u_y) [, (u_z)],   u = alpha L v
//   b-chain (fp32):  (b_x + i b_y) [, (b_z)]      -> p = -(alpha L~)^{-1} b  (same packing)
//   Leray b-chain:   b_c + i 0 (c < d)            -> (b_Lx + i b_Ly), (b_Lz), (p_x + i p_y), (p_z)
//   Leray v-chain:   v_c + i 0 (c < d)            -> (u_x + i u_y), (u_z),  u = alpha L P_L v
// Packing two real fields as A + iB is exact for real even multipliers (alpha L, its
// inverse); the Leray outputs are packed after projection from the per-component spectra.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.cuh"
#include "rfft.cuh"
#include "tma.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>

namespace topt {

void upload_twiddles() {
  static float2 hf[2048];
  static double2 hd[2048];
  for (int N = 4; N <= 1024; N *= 2)
    for (int m = 0; m < N; ++m) {
      const double a = -2.0 * M_PI * (double)m / (double)N;
      hd[N + m] = make_double2(cos(a), sin(a));
      hf[N + m] = make_float2((float)cos(a), (float)sin(a));
    }
  cudaMemcpyToSymbol(g_twiddle, hf, sizeof(hf));
  cudaMemcpyToSymbol(g_twiddle_d, hd, sizeof(hd));
}

__device__ __forceinline__ float kfreq(int q, int N) { return (float)(q <= N / 2 ? q : q - N); }
__device__ __forceinline__ float kprime(int q, int N) {  // Nyquist zeroed (R3)
  return q == N / 2 ? 0.0f : kfreq(q, N);
}

// values per thread: fp32 lines 16 (radix 16), fp64 lines and multi-field fp32 lines 8
template <int N, int EMAX> struct Ev { static constexpr int v = N < EMAX ? N : EMAX; };
// strided derivative lines: radix 16 (one smem exchange at N = 256) when summing time
// slices, radix 8 (two exchanges, ~110 registers: 2 resident blocks instead of 1) for a
// single field, where latency hiding needs the occupancy

static int num_sms() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// persistent grid: resident blocks of `kern`, capped by the number of work items
// resident blocks per SM of (kernel, threads, smem), queried once (host API calls are
// microseconds each: at small grids they would dominate the launch path)
template <typename K>
static int resident_per_sm(K kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  static std::map<const void*, size_t> smem_set;  // the attribute only ever grows per kernel
  const auto key = std::make_tuple((const void*)kern, threads, smem);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  size_t& cur = smem_set[(const void*)kern];
  if (smem > cur) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cur = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  cache[key] = per_sm;
  return per_sm;
}

template <typename K>
static int persistent_blocks(K kern, int threads, size_t smem, long long items) {
  const int per_sm = resident_per_sm(kern, threads, smem);
  long long b = (long long)num_sms() * per_sm;
  if (b > items) b = items;
  if (b < 1) b = 1;
  return (int)b;
}

// =====================================================================================
// Derivative / body-force accumulation along x (contiguous lines).  Two real lines are
// packed into one complex line; the odd multiplier i k' maps real to real (R3), so
// IFFT(i k' FFT(a + i b)) = d a + i d b.   out = beta out + sum_j w_j lam_j d psi_j.
// =====================================================================================
template <int N>
__global__ void __launch_bounds__(kThreads) k_rdx(Geom g, const float* __restrict__ psi, size_t psi_stride,
                                                  const float* __restrict__ lam, size_t lam_stride, DerivWeights w,
                                                  int J, float beta, float* __restrict__ out, int ngroups) {
  constexpr int E = Ev<N, 16>::v, T = N / E, LPB = kThreads / T;
  constexpr bool WARP = T <= 32;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) float2 smem[];
  const int line = threadIdx.x / T, t = threadIdx.x % T;
  float2* lbuf = smem + line * R::STRIDE;
  float2 tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const size_t nreal = (size_t)g.ny * g.nz;
  const float invN = 1.0f / (float)N;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const size_t la = ((size_t)grp * LPB + line) * 2;  // real lines la, la + 1
    const bool ok = la < nreal;
    const size_t oa = la * N + t, ob = oa + N;
    float acc0[E], acc1[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc0[e] = acc1[e] = 0.0f;
    for (int j = 0; j < J; ++j) {
      const float* src = psi + j * psi_stride;
      float2 z[E];
#pragma unroll
      for (int e = 0; e < E; ++e)
        z[e] = ok ? make_float2(__ldg(src + oa + T * e), __ldg(src + ob + T * e)) : make_float2(0.f, 0.f);
      rf_fft<N, E, false, WARP>(z, lbuf, t, tw);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float k = kprime(t + T * e, N) * invN;
        z[e] = make_float2(-k * z[e].y, k * z[e].x);  // i k' z / N
      }
      rf_fft<N, E, true, WARP>(z, lbuf, t, tw);
      const float wj = w.w[j];
      if (lam) {
        const float* lj = lam + j * lam_stride;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float l0 = ok ? __ldg(lj + oa + T * e) : 0.f, l1 = ok ? __ldg(lj + ob + T * e) : 0.f;
          acc0[e] = fmaf(wj * l0, z[e].x, acc0[e]);
          acc1[e] = fmaf(wj * l1, z[e].y, acc1[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          acc0[e] = fmaf(wj, z[e].x, acc0[e]);
          acc1[e] = fmaf(wj, z[e].y, acc1[e]);
        }
      }
    }
    if (ok) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float r0 = acc0[e], r1 = acc1[e];
        if (beta != 0.0f) {
          r0 += beta * out[oa + T * e];
          r1 += beta * out[ob + T * e];
        }
        out[oa + T * e] = r0;
        out[ob + T * e] = r1;
      }
    }
  }
}

// =====================================================================================
// Derivative / body-force accumulation along a strided axis (y or z).  A work item is a
// tile of 2*TXC consecutive x columns x N positions; columns (2c, 2c+1) share a complex
// line.  Thread (c, t), c fastest: every load / store of a row is one contiguous
// 8*TXC-byte segment.
// =====================================================================================
#ifndef TOPT_RDS16_MINB
#define TOPT_RDS16_MINB 2
#endif
template <int N, int EMAX>
__global__ void __launch_bounds__(kThreads, (EMAX == 8 || N == 256 ? TOPT_RDS16_MINB : 1)) k_rds(Geom g, int axis, int TXC,
                                                                       const float* __restrict__ psi,
                                                                       size_t psi_stride, const float* __restrict__ lam,
                                                                       size_t lam_stride, DerivWeights w, int J,
                                                                       float beta, float* __restrict__ out, int nitems) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) float2 smem[];
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  float2* lbuf = smem + c * R::STRIDE;
  float2 tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / (2 * TXC);
  const unsigned S = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
  const float invN = 1.0f / (float)N;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
    const unsigned base = (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0 + 2 * c;
    float2 acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
    for (int j = 0; j < J; ++j) {
      const float* src = psi + j * psi_stride;
      float2 z[E];
#pragma unroll
      for (int e = 0; e < E; ++e) z[e] = __ldg(reinterpret_cast<const float2*>(src + base + (t + T * e) * S));
      rf_fft<N, E, false, false>(z, lbuf, t, tw);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float k = kprime(t + T * e, N) * invN;
        z[e] = make_float2(-k * z[e].y, k * z[e].x);
      }
      rf_fft<N, E, true, false>(z, lbuf, t, tw);
      const float wj = w.w[j];
      if (lam) {
        const float* lj = lam + j * lam_stride;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float2 l = __ldg(reinterpret_cast<const float2*>(lj + base + (t + T * e) * S));
          acc[e].x = fmaf(wj * l.x, z[e].x, acc[e].x);
          acc[e].y = fmaf(wj * l.y, z[e].y, acc[e].y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          acc[e].x = fmaf(wj, z[e].x, acc[e].x);
          acc[e].y = fmaf(wj, z[e].y, acc[e].y);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      float2* o = reinterpret_cast<float2*>(out + base + (t + T * e) * S);
      float2 r = acc[e];
      if (beta != 0.0f) {
        const float2 p = *o;
        r.x += beta * p.x;
        r.y += beta * p.y;
      }
      *o = r;
    }
  }
}

// z-slabs, P2P transport: the z pass of the body force fused with both transposes.  The block
// works on the y-slab rows of its rank (geometry gy: nz = global planes, ny = this rank's rows,
// ky0 = their global offset) but reads every z-line element straight from the z-slab of the
// rank owning that plane (pointer tables: rank q's slice-0 psi / lam, local or peer-mapped), and
// writes b_z back into the owners' z-slabs — no y-slab copies of the 2(S+1) slices, no return
// transpose.  Same arithmetic as k_rds (axis 2).
struct ZTab {
  const float* psi[8];
  const float* lam[8];
  float* out[8];
};
template <int N, int EMAX>
__global__ void __launch_bounds__(kThreads, (EMAX == 8 || N == 256 ? TOPT_RDS16_MINB : 1)) k_rds_zpull(
    Geom g, int TXC, ZTab tb, size_t psi_stride, size_t lam_stride, int lnzl, unsigned plane_src, DerivWeights w,
    int J, int nitems) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) float2 smem[];
  __shared__ const float* sps[8];
  __shared__ const float* sls[8];
  __shared__ float* sos[8];
  if (threadIdx.x < 8) {
    sps[threadIdx.x] = tb.psi[threadIdx.x];
    sls[threadIdx.x] = tb.lam[threadIdx.x];
    sos[threadIdx.x] = tb.out[threadIdx.x];
  }
  __syncthreads();
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  float2* lbuf = smem + c * R::STRIDE;
  float2 tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / (2 * TXC);
  const float invN = 1.0f / (float)N;
  const int zmask = (1 << lnzl) - 1;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
    const unsigned yx = ((unsigned)(g.ky0 + outer) << g.lx) + x0 + 2 * c;  // (y, x) in a source plane
    float2 acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
    for (int j = 0; j < J; ++j) {
      float2 z[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int zr = t + T * e;
        z[e] = __ldcv(reinterpret_cast<const float2*>(sps[zr >> lnzl] + j * psi_stride + (zr & zmask) * plane_src + yx));
      }
      rf_fft<N, E, false, false>(z, lbuf, t, tw);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float k = kprime(t + T * e, N) * invN;
        z[e] = make_float2(-k * z[e].y, k * z[e].x);
      }
      rf_fft<N, E, true, false>(z, lbuf, t, tw);
      const float wj = w.w[j];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int zr = t + T * e;
        const float2 l = __ldcv(reinterpret_cast<const float2*>(sls[zr >> lnzl] + j * lam_stride + (zr & zmask) * plane_src + yx));
        acc[e].x = fmaf(wj * l.x, z[e].x, acc[e].x);
        acc[e].y = fmaf(wj * l.y, z[e].y, acc[e].y);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int zr = t + T * e;
      *reinterpret_cast<float2*>(sos[zr >> lnzl] + (zr & zmask) * plane_src + yx) = acc[e];
    }
  }
  __threadfence_system();  // the b_z stores into the peers' slabs, before the barrier that follows
}

static int ilog2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

template <int N>
static void zpull_launch(const Geom& gy, const ZTab& tb, size_t psi_stride, size_t lam_stride, int nzl,
                         unsigned plane_src, const DerivWeights& w, int J, cudaStream_t st) {
  constexpr int EMAX = 16;
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  int TXC = kThreads / T;
  if (2 * TXC > gy.nx) TXC = gy.nx / 2;
  const int threads = TXC * T;
  const size_t sm = (size_t)TXC * R::STRIDE * sizeof(float2);
  const long long items = (long long)(gy.nx / (2 * TXC)) * gy.ny;
  const int blocks = persistent_blocks(k_rds_zpull<N, EMAX>, threads, sm, items);
  k_rds_zpull<N, EMAX><<<blocks, threads, sm, st>>>(gy, TXC, tb, psi_stride, lam_stride, ilog2i(nzl), plane_src, w,
                                                    J, (int)items);
  count_launch();
}

// Body force along a strided axis (J time slices): as k_rds, but the psi tile of slice j+1
// and the lam tile of slice j are copied global -> shared with cp.async while slice j is
// transformed, so the HBM latency of both streams hides behind the line FFTs (no extra
// registers).  Tiles are [N rows][TXC column pairs] (8*TXC bytes per row).
__device__ __forceinline__ void cp_async16_f(void* smem, const float* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit_f() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1_f() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait0_f() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int N, int EMAX>
__global__ void __launch_bounds__(kThreads, (N == 256 ? TOPT_RDS16_MINB : 1)) k_rds_pf(
    Geom g, int axis, int TXC, const float* __restrict__ psi, size_t psi_stride, const float* __restrict__ lam,
    size_t lam_stride, DerivWeights w, int J, float beta, float* __restrict__ out, int nitems) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) float2 smem[];
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  float2* lbuf = smem + c * R::STRIDE;
  float2* Pt = smem + TXC * R::STRIDE;  // psi tile
  float2* Lt = Pt + N * TXC;            // lam tile
  float2 tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / (2 * TXC);
  const unsigned S = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
  const float invN = 1.0f / (float)N;
  const int half = TXC / 2, nchunk = N * half;  // 16-byte chunks per tile
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
    const unsigned tile0 = (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0;
    const unsigned base = tile0 + 2 * c;
    auto issue = [&](float2* dst, const float* field) {
      for (int i = threadIdx.x; i < nchunk; i += blockDim.x) {
        const int row = i / half, k = i % half;
        cp_async16_f(dst + row * TXC + 2 * k, field + tile0 + row * S + 4 * k);
      }
    };
    float2 acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
    issue(Pt, psi);
    cp_commit_f();
    for (int j = 0; j < J; ++j) {
      if (lam) issue(Lt, lam + j * lam_stride);
      cp_commit_f();
      cp_wait1_f();  // psi_j has landed (lam_j may be in flight)
      __syncthreads();
      float2 z[E];
#pragma unroll
      for (int e = 0; e < E; ++e) z[e] = Pt[(t + T * e) * TXC + c];
      __syncthreads();  // the psi tile is free
      if (j + 1 < J) issue(Pt, psi + (j + 1) * psi_stride);
      cp_commit_f();
      rf_fft<N, E, false, false>(z, lbuf, t, tw);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float k = kprime(t + T * e, N) * invN;
        z[e] = make_float2(-k * z[e].y, k * z[e].x);
      }
      rf_fft<N, E, true, false>(z, lbuf, t, tw);
      const float wj = w.w[j];
      cp_wait1_f();  // lam_j has landed (psi_{j+1} may be in flight)
      __syncthreads();
      if (lam) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float2 l = Lt[(t + T * e) * TXC + c];
          acc[e].x = fmaf(wj * l.x, z[e].x, acc[e].x);
          acc[e].y = fmaf(wj * l.y, z[e].y, acc[e].y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          acc[e].x = fmaf(wj, z[e].x, acc[e].x);
          acc[e].y = fmaf(wj, z[e].y, acc[e].y);
        }
      }
      __syncthreads();  // the lam tile is free
    }
    cp_wait0_f();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      float2* o = reinterpret_cast<float2*>(out + base + (t + T * e) * S);
      float2 r = acc[e];
      if (beta != 0.0f) {
        const float2 p = *o;
        r.x += beta * p.x;
        r.y += beta * p.y;
      }
      *o = r;
    }
  }
}

template <int N, int EMAX>
static void rds_pf_launch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w, cudaStream_t st) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  int TXC = kThreads / T;
  if (2 * TXC > g.nx) TXC = g.nx / 2;
  const int threads = TXC * T;
  const size_t sm = ((size_t)TXC * R::STRIDE + 2 * (size_t)N * TXC) * sizeof(float2);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / (2 * TXC)) * outer;
  const int blocks = persistent_blocks(k_rds_pf<N, EMAX>, threads, sm, items);
  k_rds_pf<N, EMAX><<<blocks, threads, sm, st>>>(g, axis, TXC, a.psi, a.psi_stride, a.lam, a.lam_stride, w, a.J,
                                                 a.beta, a.out, (int)items);
}

// =====================================================================================
// Body-force accumulation along a strided axis with TMA staging (k_rds_tma).  Same arithmetic
// and thread layout as k_rds (thread (c, t), c fastest; TXC = kThreads / T columns of complex
// pairs), but the slice tiles psi_j and lam_j — N positions x 2 TXC floats — are brought in by
// TMA TENSOR copies (one per 256 positions and field, issued by one thread, completing on the
// slot's mbarrier) ONE SLICE AHEAD into a two-slot ring, so the next slice streams in while the
// current one is transformed, with no registers spent on the prefetch.  The tensor maps view
// the S+1 slices as a 4D tensor (x, y, z, slice).  The psi tile doubles as the FFT exchange
// scratch once its values are in registers (interleaved [position][column] layout,
// conflict-free: a warp's 16 columns x 2 positions are 32 consecutive complex words).  The
// (item, slice) sequence of a persistent block is pipelined across items.
// =====================================================================================
struct TmaDeriv {
  CUtensorMap psi, lam;  // 4D (x, y, z, slice), box (2 TXC, N or 1, 1 or N, 1) capped at 256 positions
};
#ifndef TOPT_RDS_TMA_THREADS
#define TOPT_RDS_TMA_THREADS 128  // block size: 128 threads, 64 KB of tiles, 3 blocks per SM (256: 1 block, -6%)
#endif
constexpr int kRdsThreads = TOPT_RDS_TMA_THREADS;
template <int N>
__global__ void __launch_bounds__(kRdsThreads, kRdsThreads == 256 ? 1 : 3) k_rds_tma(
    Geom g, int axis, const __grid_constant__ TmaDeriv tm, bool has_lam, DerivWeights w, int J, float beta,
    float* __restrict__ out, int nitems) {
  constexpr int E = Ev<N, 16>::v, T = N / E, TXC = kRdsThreads / T;
  constexpr int TILE = N * 2 * TXC;  // floats per staged tile
  constexpr int BOX = N < 256 ? N : 256;
  extern __shared__ __align__(128) float smf[];
  float* tiles = smf;                                            // [slot][psi, lam][N][2 TXC]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smf + 4 * TILE);  // one per slot
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  float2 tw[RfCfg<N, E>::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / (2 * TXC);
  const size_t S = axis == 1 ? (size_t)g.nx : (size_t)g.nx * g.ny;
  const float invN = 1.0f / (float)N;
  const int nmine = blockIdx.x < nitems ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total = nmine * J;
  // thread 0: stage slice k of this block's sequence (item blockIdx.x + (k / J) gridDim.x, slice k % J)
  auto issue = [&](int k) {
    const int slot = k & 1, item = blockIdx.x + (k / J) * gridDim.x, j = k % J;
    const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
    float* dp = tiles + (2 * slot) * TILE;
    tma::mbar_arrive_expect_tx(bars + slot, (has_lam ? 2u : 1u) * TILE * 4u);
    for (int p0 = 0; p0 < N; p0 += BOX) {
      const int cy = axis == 1 ? p0 : outer, cz = axis == 1 ? outer : p0;
      tma::tensor4_g2s(dp + p0 * 2 * TXC, &tm.psi, x0, cy, cz, j, bars + slot);
      if (has_lam) tma::tensor4_g2s(dp + TILE + p0 * 2 * TXC, &tm.lam, x0, cy, cz, j, bars + slot);
    }
  };
  if (threadIdx.x == 0) {
    tma::mbar_init(bars, 1);
    tma::mbar_init(bars + 1, 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && total > 0) issue(0);
  float2 acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
  for (int k = 0; k < total; ++k) {
    const int slot = k & 1, j = k % J;
    // slot (k+1)&1 held slice k-1: every thread left it at the end-of-slice barrier below
    TOPT_STRESS_POINT(k * 5 + 31);
    if (threadIdx.x == 0 && k + 1 < total) issue(k + 1);
    TOPT_STRESS_POINT(k * 5 + 32);
    tma::mbar_wait(bars + slot, (unsigned)(k >> 1) & 1u);
    float2* tp = reinterpret_cast<float2*>(tiles + (2 * slot) * TILE);
    const float2* tl = reinterpret_cast<const float2*>(tiles + (2 * slot + 1) * TILE);
    float2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) z[e] = tp[(t + T * e) * TXC + c];
    __syncthreads();  // the psi tile becomes the exchange scratch
    rf_fft<N, E, false, false, false, TXC>(z, tp + c, t, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float kk = kprime(t + T * e, N) * invN;
      z[e] = make_float2(-kk * z[e].y, kk * z[e].x);
    }
    rf_fft<N, E, true, false, false, TXC>(z, tp + c, t, tw);
    const float wj = w.w[j];
    if (has_lam) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float2 l = tl[(t + T * e) * TXC + c];
        acc[e].x = fmaf(wj * l.x, z[e].x, acc[e].x);
        acc[e].y = fmaf(wj * l.y, z[e].y, acc[e].y);
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        acc[e].x = fmaf(wj, z[e].x, acc[e].x);
        acc[e].y = fmaf(wj, z[e].y, acc[e].y);
      }
    }
    if (j == J - 1) {
      const int item = blockIdx.x + (k / J) * gridDim.x;
      const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
      const size_t b0 = (axis == 1 ? ((size_t)outer << (g.lx + g.ly)) : ((size_t)outer << g.lx)) + x0 + 2 * c;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float2* o = reinterpret_cast<float2*>(out + b0 + (t + T * e) * S);
        float2 r = acc[e];
        if (beta != 0.0f) {
          const float2 p = *o;
          r.x += beta * p.x;
          r.y += beta * p.y;
        }
        *o = r;
        acc[e] = make_float2(0.f, 0.f);
      }
    }
    TOPT_STRESS_POINT(k * 5 + 33);
    __syncthreads();  // slot k&1 (tiles and scratch) free for slice k+2
  }
}

#ifndef TOPT_RDS_TMA
#define TOPT_RDS_TMA 1
#endif
#ifndef TOPT_RDS_TMA_J1
#define TOPT_RDS_TMA_J1 0  // 1: div v passes TMA-staged too (measured slower: 1.63 vs 2.09 TB/s)
#endif
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
// 4D map of the slices of a field: dims (nx, ny, nz, J), slice stride `stride` floats
static bool slice_map(CUtensorMap* m, const float* base, const Geom& g, size_t stride, int J, int axis, int box_x,
                      int box_n) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz, (cuuint64_t)J};
  const cuuint64_t strides[3] = {(cuuint64_t)g.nx * 4, (cuuint64_t)g.nx * g.ny * 4, (cuuint64_t)stride * 4};
  const cuuint32_t box[4] = {(cuuint32_t)box_x, (cuuint32_t)(axis == 1 ? box_n : 1), (cuuint32_t)(axis == 1 ? 1 : box_n),
                             1u};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int N>
static bool rds_tma_launch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w, cudaStream_t st) {
  constexpr int T = N / Ev<N, 16>::v, TXC = kRdsThreads / T;
  if (!TOPT_RDS_TMA || N < 128 || N > 1024 || 2 * TXC > g.nx || g.nx % (2 * TXC) || 2 * TXC * 4 < 16) return false;
  if (((uintptr_t)a.psi | (uintptr_t)(a.lam ? a.lam : a.psi)) & 15) return false;
  if ((a.psi_stride | (a.lam ? a.lam_stride : 0)) & 3) return false;
  TmaDeriv tm{};
  const int box_n = N < 256 ? N : 256;
  if (!slice_map(&tm.psi, a.psi, g, a.psi_stride, a.J, axis, 2 * TXC, box_n)) return false;
  if (a.lam && !slice_map(&tm.lam, a.lam, g, a.lam_stride, a.J, axis, 2 * TXC, box_n)) return false;
  const size_t sm = 4 * (size_t)N * 2 * TXC * sizeof(float) + 2 * sizeof(uint64_t);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / (2 * TXC)) * outer;
  const int blocks = persistent_blocks(k_rds_tma<N>, kRdsThreads, sm, items);
  k_rds_tma<N><<<blocks, kRdsThreads, sm, st>>>(g, axis, tm, a.lam != nullptr, w, a.J, a.beta, a.out, (int)items);
  return true;
}

template <int N, int EMAX>
static void rds_launch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w, cudaStream_t st) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  using R = RfCfg<N, E>;
  int TXC = kThreads / T;
  if (2 * TXC > g.nx) TXC = g.nx / 2;
  const int threads = TXC * T;
  const size_t sm = (size_t)TXC * R::STRIDE * sizeof(float2);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / (2 * TXC)) * outer;
  const int blocks = persistent_blocks(k_rds<N, EMAX>, threads, sm, items);
  k_rds<N, EMAX><<<blocks, threads, sm, st>>>(g, axis, TXC, a.psi, a.psi_stride, a.lam, a.lam_stride, w, a.J, a.beta,
                                              a.out, (int)items);
}

// Single-field pass (div v: J = 1, no lam): k_rds with the next item's line elements (and the
// accumulator it updates) loaded into registers while the current item is transformed — one item
// holds too few bytes in flight to cover the HBM latency at two resident blocks per SM.
#ifndef TOPT_RDS1
#define TOPT_RDS1 1
#endif
template <int N>
__global__ void __launch_bounds__(kThreads, 2) k_rds1(Geom g, int axis, int TXC, const float* __restrict__ psi,
                                                   float w0, float beta, float* __restrict__ out, int nitems) {
  constexpr int E = Ev<N, 8>::v, T = N / E;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) float2 smem[];
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  float2* lbuf = smem + c * R::STRIDE;
  float2 tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / (2 * TXC);
  const unsigned S = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
  const float invN = 1.0f / (float)N;
  auto base_of = [&](int item) -> unsigned {
    const int x0 = (item % tilesx) * 2 * TXC, outer = item / tilesx;
    return (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0 + 2 * c;
  };
  float2 zn[E], on[E];
  auto fetch = [&](int item) {
    const unsigned b = base_of(item);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      zn[e] = __ldg(reinterpret_cast<const float2*>(psi + b + (t + T * e) * S));
      on[e] = beta != 0.0f ? *reinterpret_cast<const float2*>(out + b + (t + T * e) * S) : make_float2(0.f, 0.f);
    }
  };
  if ((int)blockIdx.x < nitems) fetch(blockIdx.x);
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    float2 z[E], o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      z[e] = zn[e];
      o[e] = on[e];
    }
    if (item + (int)gridDim.x < nitems) fetch(item + gridDim.x);
    rf_fft<N, E, false, false>(z, lbuf, t, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float k = kprime(t + T * e, N) * invN;
      z[e] = make_float2(-k * z[e].y, k * z[e].x);
    }
    rf_fft<N, E, true, false>(z, lbuf, t, tw);
    const unsigned b = base_of(item);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      float2 r = make_float2(fmaf(w0, z[e].x, 0.f), fmaf(w0, z[e].y, 0.f));
      if (beta != 0.0f) {
        r.x += beta * o[e].x;
        r.y += beta * o[e].y;
      }
      *reinterpret_cast<float2*>(out + b + (t + T * e) * S) = r;
    }
  }
}
template <int N>
static void rds1_launch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w, cudaStream_t st) {
  constexpr int E = Ev<N, 8>::v, T = N / E;
  using R = RfCfg<N, E>;
  int TXC = kThreads / T;
  if (2 * TXC > g.nx) TXC = g.nx / 2;
  const int threads = TXC * T;
  const size_t sm = (size_t)TXC * R::STRIDE * sizeof(float2);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / (2 * TXC)) * outer;
  const int blocks = persistent_blocks(k_rds1<N>, threads, sm, items);
  k_rds1<N><<<blocks, threads, sm, st>>>(g, axis, TXC, a.psi, w.w[0], a.beta, a.out, (int)items);
}

template <int N>
static void deriv_dispatch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w, cudaStream_t st) {
  if (axis == 0) {
    constexpr int E = Ev<N, 16>::v, T = N / E;
    using R = RfCfg<N, E>;
    constexpr int LPB = kThreads / T;
    const size_t sm = (size_t)LPB * R::STRIDE * sizeof(float2);
    const size_t nreal = (size_t)g.ny * g.nz;
    const long long groups = (long long)((nreal + 2 * LPB - 1) / (2 * LPB));
    const int blocks = persistent_blocks(k_rdx<N>, kThreads, sm, groups);
    k_rdx<N><<<blocks, kThreads, sm, st>>>(g, a.psi, a.psi_stride, a.lam, a.lam_stride, w, a.J, a.beta, a.out,
                                            (int)groups);
  } else if (a.J == 1) {
    // single field (div v): the TMA-staged pass pipelines across work items; else occupancy first
    if (TOPT_RDS_TMA_J1 && rds_tma_launch<N>(g, axis, a, w, st)) {
    } else if (TOPT_RDS1 && !a.lam) {
      rds1_launch<N>(g, axis, a, w, st);
    } else {
      rds_launch<N, 8>(g, axis, a, w, st);
    }
  } else {
    // time-slice sums: one smem exchange per FFT; at N >= 512 (one resident block per SM)
    // the tiles of the next slice are prefetched with cp.async (measured: +7% at 512^3,
    // -10% at 256^3 where two blocks per SM already overlap the loads)
    if (rds_tma_launch<N>(g, axis, a, w, st)) {
    } else if constexpr (N >= 512) {
      rds_pf_launch<N, 16>(g, axis, a, w, st);
    } else {
      rds_launch<N, 16>(g, axis, a, w, st);
    }
  }
  count_launch();
}

#define TOPT_DISPATCH_N(NV, FN, ...)                   \
  switch (NV) {                                        \
    case 8: FN<8>(__VA_ARGS__); break;                 \
    case 16: FN<16>(__VA_ARGS__); break;               \
    case 32: FN<32>(__VA_ARGS__); break;               \
    case 64: FN<64>(__VA_ARGS__); break;               \
    case 128: FN<128>(__VA_ARGS__); break;             \
    case 256: FN<256>(__VA_ARGS__); break;             \
    case 512: FN<512>(__VA_ARGS__); break;             \
    case 1024: FN<1024>(__VA_ARGS__); break;           \
    default: fprintf(stderr, "topt: unsupported N %d\n", NV); \
  }

void launch_deriv_zpull(const Geom& gy, const float* const* psi, const float* const* lam, float* const* out, int P,
                        size_t psi_stride, size_t lam_stride, int nzl, size_t plane_src, const double* wts, int J,
                        cudaStream_t st) {
  ZTab tb{};
  for (int q = 0; q < P && q < 8; ++q) {
    tb.psi[q] = psi[q];
    tb.lam[q] = lam[q];
    tb.out[q] = out[q];
  }
  DerivWeights w;
  for (int j = 0; j < J && j < kMaxWeights; ++j) w.w[j] = (float)wts[j];
  TOPT_DISPATCH_N(gy.nz, zpull_launch, gy, tb, psi_stride, lam_stride, nzl, (unsigned)plane_src, w, J, st);
}

void launch_deriv_accum(const Geom& g, int axis, const DerivArgs& a, cudaStream_t st) {
  DerivWeights w;
  for (int j = 0; j < a.J && j < kMaxWeights; ++j) w.w[j] = (float)a.w[j];
  const int N = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  TOPT_DISPATCH_N(N, deriv_dispatch, g, axis, a, w, st);
}

// =====================================================================================
// Preconditioner / regulariser chains: 3D FFT = x pass, [y pass], last-axis pass with the
// fused spectral operator, [y^-1], x^-1 (fused into the assembly for the b-chain).
//   v-chain (fp64 arithmetic AND fp64 intermediates): u = alpha L v.  L = |k|^{2p}
//   amplifies any rounding at high |k| by up to (k_max/k)^{2p}, so the chain that applies
//   it runs in double.
//   b-chain (fp32): the smoothing inverse -(alpha L~)^{-1} and the Leray projector are
//   well conditioned.  Leray outputs b_L and p are separate pairs — never one complex
//   field, whose parts differ by up to 1/alpha and would pollute each other in fp32.
// =====================================================================================
template <typename C>
struct ZList { C* z[4]; };
struct RealIn { const float* re[3]; const float* im[3]; };
struct RealOut { float* re[3]; float* im[3]; };

// x pass forward: Z_f[row][q] = FFT_x(re_f + i im_f)[q]; blockIdx.y = field f
template <int N, int EMAX, typename C>
__global__ void __launch_bounds__(kThreads) k_rx_fwd(Geom g, RealIn in, ZList<C> Z, int ngroups) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E, LPB = kThreads / T;
  constexpr bool WARP = T <= 32;
  using R = RfCfg<N, E>;
  using Tr = typename Real<C>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int line = threadIdx.x / T, t = threadIdx.x % T;
  C* lbuf = reinterpret_cast<C*>(smraw) + line * R::STRIDE;
  C tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const size_t nrows = (size_t)g.ny * g.nz;
  const int f = blockIdx.y;
  const float* re = in.re[f];
  const float* im = in.im[f];
  C* Zf = Z.z[f];
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const size_t row = (size_t)grp * LPB + line;
    const bool ok = row < nrows;
    const size_t o = row * N + t;
    C a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float x = (ok && re) ? __ldg(re + o + T * e) : 0.f;
      const float y = (ok && im) ? __ldg(im + o + T * e) : 0.f;
      a[e] = mk((Tr)x, (Tr)y);
    }
    rf_fft<N, E, false, WARP>(a, lbuf, t, tw);
    if (ok) {
#pragma unroll
      for (int e = 0; e < E; ++e) Zf[o + T * e] = a[e];
    }
  }
}

// x pass inverse to real outputs: re_f + i im_f = IFFT_x(Z_f)  (either output may be null)
template <int N, int EMAX, typename C>
__global__ void __launch_bounds__(kThreads) k_rx_inv(Geom g, ZList<C> Z, RealOut out, int ngroups) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E, LPB = kThreads / T;
  constexpr bool WARP = T <= 32;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int line = threadIdx.x / T, t = threadIdx.x % T;
  C* lbuf = reinterpret_cast<C*>(smraw) + line * R::STRIDE;
  C tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const size_t nrows = (size_t)g.ny * g.nz;
  const int f = blockIdx.y;
  const C* Zf = Z.z[f];
  float* re = out.re[f];
  float* im = out.im[f];
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const size_t row = (size_t)grp * LPB + line;
    const bool ok = row < nrows;
    const size_t o = row * N + t;
    C a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = ok ? Zf[o + T * e] : mk((typename Real<C>::T)0, (typename Real<C>::T)0);
    rf_fft<N, E, true, WARP>(a, lbuf, t, tw);
    if (ok) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (re) re[o + T * e] = (float)a[e].x;
        if (im) im[o + T * e] = (float)a[e].y;
      }
    }
  }
}

// Strided-axis pass (lines along y in 3D, along the last axis otherwise).  A work item is
// TXC consecutive complex columns; thread (c, t), c fastest.
//   MODE 0: forward FFT only        (3D y pass)
//   MODE 1: inverse FFT only        (3D y^-1 pass)
//   MODE 2: fwd, Z *= alpha L(k)/n, inv                        (v-chain, last axis)
//   MODE 3: fwd, Z *= -1/(alpha L~(k) n), inv                  (b-chain, last axis)
//   MODE 4: fwd, Leray + inverse regulariser, inv; d -> 2 (2D) / 4 (3D) fields (b-chain)
//   MODE 5: fwd, alpha L P_L, inv; d -> 1 (2D) / 2 (3D) fields (incompressible v-chain)
// Modes 0-3 take one field per item (item = tile + field * tiles); modes 4/5 hold the d
// component spectra of a tile in registers at once.
struct SpecOp {
  double alpha;
  int p;
  double invn;
};

__device__ __forceinline__ double regL(double kk, int p) { return p == 1 ? kk : (p == 2 ? kk * kk : kk * kk * kk); }

// z-slabs, P2P transport: the last-axis pass of a single-field mode (MODE <= 3) run in place on
// the distributed z-slabs — element (z, y, x) of field f lives in rank z / nzl's slab at plane
// z % nzl (tab[f][q]: rank q's field base, local or peer-mapped) — so neither transpose exists.
struct RemoteZ {
  int lnzl;            // log2 of the planes per rank
  unsigned plane_src;  // elements per z-slab plane (nx * global ny)
  const void* tab[4][8];
};
template <int N, int EMAX, int MODE, typename C, bool REM = false>
__global__ void __launch_bounds__(kThreads, (MODE >= 4 ? 1 : 2)) k_rstrided(Geom g, int axis, int TXC, int NIN, int NOUT, ZList<C> Z,
                                                       SpecOp op, int nitems, RemoteZ rz = RemoteZ{}) {
  static_assert(!REM || MODE <= 3, "remote addressing: single-field modes");
  __shared__ C* rtab[REM ? 32 : 1];
  if constexpr (REM) {
    if (threadIdx.x < 32) rtab[threadIdx.x] = (C*)rz.tab[threadIdx.x >> 3][threadIdx.x & 7];
    __syncthreads();
  }
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  constexpr int NF = MODE >= 4 ? 3 : 1;  // fields held in registers
  using R = RfCfg<N, E>;
  using Tr = typename Real<C>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  C* lbuf = reinterpret_cast<C*>(smraw) + c * R::STRIDE;
  C tw[R::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / TXC;
  const int outerN = axis == 1 ? g.nz : g.ny;
  const int tiles = tilesx * outerN;
  const unsigned Su = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int tt = item % tiles;
    const int f0 = MODE >= 4 ? 0 : item / tiles;
    const int x0 = (tt % tilesx) * TXC, outer = tt / tilesx;
    const unsigned base = (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0 + c;
    // wavenumbers of this column (x) and of the outer index (3D: y)
    const int qx = x0 + c;
    const double kx = qx <= g.nx / 2 ? qx : qx - g.nx, kxp = qx == g.nx / 2 ? 0.0 : kx;
    double ky = 0.0, kyp = 0.0;
    if (g.d == 3) {
      const int nyg = g.nyg ? g.nyg : g.ny;  // y-slab layout: global row = ky0 + local row
      const int qy = outer + g.ky0;
      ky = qy <= nyg / 2 ? qy : qy - nyg;
      kyp = qy == nyg / 2 ? 0.0 : ky;
    }
    auto kl = [&](int q, double& kk, double& kl0, double& kl1) {  // |k|^2 and the last-axis k, k'
      const double kq = q <= N / 2 ? q : q - N, kqp = q == N / 2 ? 0.0 : kq;
      kl0 = kq;
      kl1 = kqp;
      kk = g.d == 3 ? kx * kx + ky * ky + kq * kq : kx * kx + kq * kq;
    };
    if constexpr (MODE <= 3) {
      C a[E];
      const C* src = Z.z[f0];
      // remote: (y, x) offset inside a z-slab plane and the owner / plane of row zr
      const unsigned yx = REM ? ((unsigned)(outer + g.ky0) << g.lx) + x0 + c : 0u;
      auto rem = [&](int zr) -> C* {
        return rtab[f0 * 8 + (zr >> rz.lnzl)] + (size_t)(zr & ((1 << rz.lnzl) - 1)) * rz.plane_src + yx;
      };
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if constexpr (REM) a[e] = __ldcv(rem(t + T * e));  // peer memory: around the local caches
        else a[e] = src[base + (t + T * e) * Su];
      }
      if constexpr (MODE != 1) rf_fft<N, E, false, false>(a, lbuf, t, tw);
      if constexpr (MODE == 2 || MODE == 3) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          double kk, k0, k1;
          kl(t + T * e, kk, k0, k1);
          const double Lk = regL(kk, op.p);
          const double Lt = Lk == 0.0 ? 1.0 : Lk;  // kernel fix
          // the smoothing multiplier in float (relative 1e-7); no fp64 division
          const Tr m = MODE == 2 ? (Tr)(op.alpha * Lk * op.invn)
                                 : (Tr)(-(float)op.invn * __frcp_rn((float)(op.alpha * Lt)));
          a[e] = mk(a[e].x * m, a[e].y * m);
        }
      }
      if constexpr (MODE != 0) rf_fft<N, E, true, false>(a, lbuf, t, tw);
      C* dst = Z.z[f0];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if constexpr (REM) *rem(t + T * e) = a[e];
        else dst[base + (t + T * e) * Su] = a[e];
      }
    } else {
      C a[NF][E];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        if (f < NIN) {
          const C* src = Z.z[f];
#pragma unroll
          for (int e = 0; e < E; ++e) a[f][e] = src[base + (t + T * e) * Su];
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) a[f][e] = mk((Tr)0, (Tr)0);
        }
      }
#pragma unroll
      for (int f = 0; f < NF; ++f)
        if (f < NIN) rf_fft<N, E, false, false>(a[f], lbuf, t, tw);
      // Leray on the d component spectra at each k (Nyquist-zeroed k', R3/R9), in place
#pragma unroll
      for (int e = 0; e < E; ++e) {
        double kk, k0, k1;
        kl(t + T * e, kk, k0, k1);
        const double kp[3] = {kxp, g.d == 3 ? kyp : k1, g.d == 3 ? k1 : 0.0};
        const double kp2 = kp[0] * kp[0] + kp[1] * kp[1] + kp[2] * kp[2];
        if (kp2 > 0.0) {
          // per-mode relative precision suffices (a 0-order projector): fp32 reciprocal
          const double ikp = (double)__frcp_rn((float)kp2);
          double dx = 0.0, dy = 0.0;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            dx += kp[f] * (double)a[f][e].x;
            dy += kp[f] * (double)a[f][e].y;
          }
          dx *= ikp;
          dy *= ikp;
#pragma unroll
          for (int f = 0; f < NF; ++f) a[f][e] = mk((Tr)((double)a[f][e].x - kp[f] * dx), (Tr)((double)a[f][e].y - kp[f] * dy));
        }
      }
      // output slots: pairs of REAL fields packed as A + iB, spectrum (Ax - By) + i (Ay + Bx)
      // 3D: 0 = (b_Lx + i b_Ly) | (u_x + i u_y), 1 = (b_Lz) | (u_z), 2 = (p_x + i p_y), 3 = (p_z)
      // 2D: 0 = (b_Lx + i b_Ly) | (u_x + i u_y), 1 = (p_x + i p_y)
      const int half = g.d == 3 ? 2 : 1;
      for (int slot = 0; slot < NOUT; ++slot) {
        const bool isp = MODE == 4 && slot >= half;
        const int s2 = slot % half;
        const int ca = 2 * s2, cb = 2 * s2 + 1 < g.d ? 2 * s2 + 1 : -1;
        C o[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          double kk, k0, k1;
          kl(t + T * e, kk, k0, k1);
          const double Lk = regL(kk, op.p);
          const double Lt = Lk == 0.0 ? 1.0 : Lk;
          const double sc = isp ? -op.invn * (double)__frcp_rn((float)(op.alpha * Lt))
                                : (MODE == 5 ? op.alpha * Lk * op.invn : op.invn);
          double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            if (f == ca) { ax = sc * (double)a[f][e].x; ay = sc * (double)a[f][e].y; }
            if (f == cb) { bx = sc * (double)a[f][e].x; by = sc * (double)a[f][e].y; }
          }
          o[e] = mk((Tr)(ax - by), (Tr)(ay + bx));
        }
        rf_fft<N, E, true, false>(o, lbuf, t, tw);
        C* dst = Z.z[slot];
#pragma unroll
        for (int e = 0; e < E; ++e) dst[base + (t + T * e) * Su] = o[e];
      }
    }
  }
  // remote (peer) stores: visible system-wide before the stream-ordered barrier that follows
  if constexpr (REM) __threadfence_system();
}

// Merged last-axis pass of the v- and b-chains (non-Leray): the forward transform of the
// v spectrum stays fp64 (the only place where rounding is amplified by alpha |k|^{2p},
// DESIGN.md §6.3); at each k the fp64 product alpha L(k) v^ is added to the b spectrum and
// the sum g^ = alpha L v^ + b^ and p^ = -b^/(alpha L~) are transformed back in fp32 — the
// inverse passes of the fp64 chain and the separate u / b reads of the assembly disappear.
// Field f of a tile: Zv[f] (fp64 (v_x + i v_y) | (v_z)), Zb[f] (fp32, same packing) ->
// G[f] = Zb[f] (g packed alike), Pp[f] (p packed alike).  Radix 8 for both precisions.
// u = alpha L v is never formed in space, so the sums the scalars need from it come from
// Parseval on the unnormalised 3D spectra (packed pairs of real fields add their |.|^2
// because the odd cross terms cancel under an even weight):
//   sum_x v.u = (1/n) sum_k alpha L |V^|^2                      -> partial slot 10
//   sum_x s.u = -(1/n) sum_k [alpha L |V^|^2 + Re(B^* V^)]_{k!=0} -> partial slot 11
// (s = -(v - vbar) + p, sum u = 0, p^ = -B^/(alpha L~)).
#ifndef TOPT_RZ_PF
#define TOPT_RZ_PF 1  // merged last-axis pass: cp.async staging of the next item's lines
#endif
#ifndef TOPT_RZ_MINB
#define TOPT_RZ_MINB 2
#endif
#ifndef TOPT_RZ_DUAL
#define TOPT_RZ_DUAL 0  // v and b forward transforms (and g, p inverse ones) in lock step (rf_fft2):
                      // 264 B of spills, bchain 4.05 -> 3.91 TB/s (also at 1 block/SM); off
#endif
template <int N>
__global__ void __launch_bounds__(kThreads, TOPT_RZ_MINB) k_rzmerge(Geom g, int axis, int TXC, ZList<double2> Zv,
                                                         ZList<float2> Zb, ZList<float2> Pp, SpecOp op, int nitems,
                                                         double* __restrict__ partials) {
  double sumVU = 0.0, sumSU = 0.0;
  constexpr int E = Ev<N, 8>::v, T = N / E;
  using R = RfCfg<N, E>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  double2* lbd = reinterpret_cast<double2*>(smraw) + c * R::STRIDE;  // fp64 line scratch
  // fp32 line scratch (same region, used after the fp64 transform).  Its column stride is chosen apart
  // from the fp64 one: at STRIDE (273 float2 = 546 words = 2 mod 32) the 8 columns of a half-warp
  // phase sit 2 words apart, exactly where the neighbouring position of the next t lands (bank
  // conflicts); TOPT_RZ_FSTRIDE float2 per column (274 = 548 words = 4 mod 32) separates them
#ifndef TOPT_RZ_FSTRIDE
#define TOPT_RZ_FSTRIDE 274
#endif
  constexpr int SF = (N == 256 && TOPT_RZ_FSTRIDE >= R::STRIDE) ? TOPT_RZ_FSTRIDE : R::STRIDE;
  static_assert(SF * sizeof(float2) <= R::STRIDE * sizeof(double2), "fp32 scratch inside the fp64 one");
  float2* lbf = reinterpret_cast<float2*>(smraw) + c * SF;
#if TOPT_RZ_DUAL
  // second fp32 scratch (its own region after the staging tiles) for the lock-step transforms
  float2* lbf2 = reinterpret_cast<float2*>(reinterpret_cast<double2*>(smraw) + TXC * R::STRIDE +
                                           (TOPT_RZ_PF ? N * TXC : 0)) +
                 (TOPT_RZ_PF ? N * TXC : 0) + c * SF;
#endif
  double2 twd[R::NTW];
  float2 twf[R::NTW];
  rf_twiddles<N, E>(twd, t);
  rf_twiddles<N, E>(twf, t);
  const int tilesx = g.nx / TXC;
  const int outerN = axis == 1 ? g.nz : g.ny;
  const int tiles = tilesx * outerN;
  const unsigned Su = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
#if TOPT_RZ_PF
  // staging tiles [N rows][TXC columns] of the fp64 v and fp32 b lines of the NEXT item,
  // filled with cp.async (16-byte chunks: one double2, or two float2) while this item's
  // lines are transformed, so the strided HBM reads overlap the fp64 FFT work
  double2* Sv = reinterpret_cast<double2*>(smraw) + TXC * R::STRIDE;
  float2* Sb = reinterpret_cast<float2*>(Sv + N * TXC);
  // TXC, tilesx and the tile count are powers of two: items and staging chunks decode by shifts.
  // Chunk i of the staging tile is (row i / TXC, column i % TXC) for v (16-byte double2) and
  // (row i / (TXC/2), columns 2 (i % (TXC/2)) + 0..1) for b; a thread's chunks are blockDim.x apart,
  // i.e. a fixed number of rows, so its source pointer advances by a constant stride.
  const int ltx = 31 - __clz(TXC), ltl = 31 - __clz(tilesx), lti = 31 - __clz(tiles);
  const size_t vstep = (size_t)(blockDim.x >> ltx) * Su, bstep = (size_t)(blockDim.x >> (ltx - 1)) * Su;
  const size_t voff = (size_t)(threadIdx.x >> ltx) * Su + (threadIdx.x & (TXC - 1));
  const size_t boff = (size_t)(threadIdx.x >> (ltx - 1)) * Su + 2 * (threadIdx.x & (TXC / 2 - 1));
  auto stage = [&](int it) {
    const int tt = it & (tiles - 1), f = it >> lti;
    const int x0 = (tt & (tilesx - 1)) << ltx, outer = tt >> ltl;
    const unsigned t0 = (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0;
    const double2* sv = Zv.z[f] + t0 + voff;
    const float2* sb = Zb.z[f] + t0 + boff;
    for (int i = threadIdx.x; i < N * TXC; i += blockDim.x, sv += vstep)
      cp_async16_f(Sv + i, reinterpret_cast<const float*>(sv));
    for (int i = threadIdx.x; i < N * TXC / 2; i += blockDim.x, sb += bstep)
      cp_async16_f(Sb + 2 * i, reinterpret_cast<const float*>(sb));
  };
  if ((int)blockIdx.x < nitems) stage(blockIdx.x);
  cp_commit_f();
#endif
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
#if TOPT_RZ_PF
    const int tt = item & (tiles - 1), f = item >> lti;
    const int x0 = (tt & (tilesx - 1)) << ltx, outer = tt >> ltl;
#else
    const int tt = item % tiles, f = item / tiles;
    const int x0 = (tt % tilesx) * TXC, outer = tt / tilesx;
#endif
    const unsigned base = (axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) : ((unsigned)outer << g.lx)) + x0 + c;
    const int qx = x0 + c;
    const double kx = qx <= g.nx / 2 ? qx : qx - g.nx;
    double ky = 0.0;
    if (g.d == 3) {
      const int nyg = g.nyg ? g.nyg : g.ny;
      const int qy = outer + g.ky0;
      ky = qy <= nyg / 2 ? qy : qy - nyg;
    }
    double2 av[E];
    float2 ab[E];
#if TOPT_RZ_PF
    // this item's lines were staged by the previous iteration (or the prologue); take them,
    // free the staging tiles and start the next item's copies before the transforms
    TOPT_STRESS_POINT(item + 41);
    cp_wait0_f();
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      av[e] = Sv[(t + T * e) * TXC + c];
      ab[e] = Sb[(t + T * e) * TXC + c];
    }
    __syncthreads();
    if (item + (int)gridDim.x < nitems) stage(item + gridDim.x);
    cp_commit_f();
#else
    const double2* sv = Zv.z[f];
    const float2* sb = Zb.z[f];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      av[e] = sv[base + (t + T * e) * Su];
      ab[e] = sb[base + (t + T * e) * Su];
    }
#endif
#if TOPT_RZ_DUAL
    rf_fft2<N, E, false, false>(av, lbd, twd, ab, lbf2, twf, t);
#else
    rf_fft<N, E, false, false>(av, lbd, t, twd);
    rf_fft<N, E, false, false>(ab, lbf, t, twf);
#endif
    float2 gg[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int q = t + T * e;
      const double kq = q <= N / 2 ? q : q - N;
      const double kk = g.d == 3 ? kx * kx + ky * ky + kq * kq : kx * kx + kq * kq;
      const double Lk = regL(kk, op.p);
      const double Lt = Lk == 0.0 ? 1.0 : Lk;  // kernel fix
      const double mu = op.alpha * Lk * op.invn;
      const double v2 = av[e].x * av[e].x + av[e].y * av[e].y;
      sumVU += op.alpha * Lk * v2;
      if (kk != 0.0) sumSU -= op.alpha * Lk * v2 + av[e].x * (double)ab[e].x + av[e].y * (double)ab[e].y;
      gg[e] = make_float2((float)(mu * av[e].x + op.invn * (double)ab[e].x),
                          (float)(mu * av[e].y + op.invn * (double)ab[e].y));
      const float mp = -(float)op.invn * __frcp_rn((float)(op.alpha * Lt));
      ab[e] = make_float2(ab[e].x * mp, ab[e].y * mp);
    }
#if TOPT_RZ_DUAL
    rf_fft2<N, E, true, false>(gg, lbf, twf, ab, lbf2, twf, t);
#else
    rf_fft<N, E, true, false>(gg, lbf, t, twf);
    rf_fft<N, E, true, false>(ab, lbf, t, twf);
#endif
    float2* dg = Zb.z[f];
    float2* dp = Pp.z[f];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      dg[base + (t + T * e) * Su] = gg[e];
      dp[base + (t + T * e) * Su] = ab[e];
    }
  }
  // block tree reduction (blockDim is a power of two, possibly < 32 at small N)
  __shared__ double red[2][kThreads];
  red[0][threadIdx.x] = sumVU;
  red[1][threadIdx.x] = sumSU;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) {
      red[0][threadIdx.x] += red[0][threadIdx.x + h];
      red[1][threadIdx.x] += red[1][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x < 2) partials[(size_t)(10 + threadIdx.x) * kMaxPartials + blockIdx.x] = red[threadIdx.x][0];
}

template <int N>
static void rzmerge_launch(const Geom& g, int axis, const ZList<double2>& Zv, const ZList<float2>& Zb,
                           const ZList<float2>& Pp, int nf, const SpecOp& op, double* partials, int* nparts,
                           cudaStream_t st) {
  constexpr int E = Ev<N, 8>::v, T = N / E;
  int TXC = kThreads / T;
  if (TXC > g.nx) TXC = g.nx;
  const int threads = TXC * T;
  size_t sm = (size_t)TXC * RfCfg<N, E>::STRIDE * sizeof(double2);
  if (TOPT_RZ_PF) sm += (size_t)N * TXC * (sizeof(double2) + sizeof(float2));  // staging tiles
  if (TOPT_RZ_DUAL) sm += (size_t)TXC * (N == 256 && TOPT_RZ_FSTRIDE >= RfCfg<N, E>::STRIDE ? TOPT_RZ_FSTRIDE : RfCfg<N, E>::STRIDE) * sizeof(float2);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / TXC) * outer * nf;
  const int blocks = persistent_blocks(k_rzmerge<N>, threads, sm, items);
  *nparts = blocks;
  k_rzmerge<N><<<blocks, threads, sm, st>>>(g, axis, TXC, Zv, Zb, Pp, op, (int)items, partials);
  count_launch();
}

// Assembly (x^-1 of the b-chain + pointwise combine), per x row (R9):
//   g = u + b_L,  s = -(v - vbar) + p,  partial sums for the scalars.
// Fields per row: non-Leray (p_x + i p_y)[, (p_z)], b_L = b from memory;
//                 Leray (b_Lx + i b_Ly)[, (b_Lz)], (p_x + i p_y)[, (p_z)].
struct AsmArgs {
  const float2* Z[4];
  const float* b;      // d*F (non-Leray)
  const float* u;      // d*F or null (0)
  const float* v;      // d*F or null (0)
  const double* vsum;  // device, d values (sum_x v_c); null => 0
  float* g;            // d*F or null
  float* s;            // d*F or null
  double* partials;    // [10][kMaxPartials]
  double ntot;         // global point count (vbar = vsum / ntot)
};

#ifndef TOPT_ASM_MINB
#define TOPT_ASM_MINB 2
#endif
#ifndef TOPT_ASM_TMA
#define TOPT_ASM_TMA 1
#endif
template <int N, int LPR, bool LERAY>
__global__ void __launch_bounds__(kThreads, TOPT_ASM_MINB) k_rassemble(Geom g, AsmArgs a, int ngroups) {
  constexpr int E = Ev<N, (LPR >= 4 ? 8 : 16)>::v, T = N / E, LPB = kThreads / T;
  constexpr bool WARP = T <= 32;
  using R = RfCfg<N, E, true>;
  extern __shared__ __align__(16) float2 smem[];
  const int line = threadIdx.x / T, t = threadIdx.x % T;
  float2* lbuf = smem + line * R::STRIDE;
  float2 tw[R::NTW];
  rf_twiddles<N, E, true>(tw, t);
  const size_t nrows = (size_t)g.ny * g.nz;
  constexpr int pf = LERAY ? LPR / 2 : 0;  // first p field
  float vbar[3] = {0.f, 0.f, 0.f};
  for (int c = 0; c < g.d; ++c) vbar[c] = a.vsum ? (float)(a.vsum[c] / a.ntot) : 0.f;
  // |g|_inf in fp32 (a max of fp32 values is exact; one FMNMX instead of a convert + fp64 compare)
  float gmax = 0.0f;
  double sgs = 0.0, svu = 0.0, ssu = 0.0, sg[3] = {0, 0, 0}, ss[3] = {0, 0, 0};
#if TOPT_ASM_TMA
  // the group's LPR spectra (LPB consecutive rows each: one contiguous chunk per field) arrive by TMA
  // bulk copies into one staging buffer, which is refilled with the NEXT group's rows as soon as
  // this group's values are in registers — the copy overlaps the transforms and the combine
  float2* stg = smem + LPB * R::STRIDE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + LPR * LPB * N);
  const bool tma_on = nrows % LPB == 0;
  auto issue = [&](int gq) {
    tma::mbar_arrive_expect_tx(bar, (unsigned)(LPR * LPB * N * sizeof(float2)));
#pragma unroll
    for (int f = 0; f < LPR; ++f)
      tma::bulk_g2s(stg + f * LPB * N, a.Z[f] + (size_t)gq * LPB * N, (unsigned)(LPB * N * sizeof(float2)), bar);
  };
  if (threadIdx.x == 0) {
    tma::mbar_init(bar, 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  if (tma_on && threadIdx.x == 0 && (int)blockIdx.x < ngroups) issue(blockIdx.x);
  unsigned phase = 0;
#endif
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const size_t row = (size_t)grp * LPB + line;
    const bool ok = row < nrows;
    const size_t o = row * N + t;
    float2 z[LPR][E];
#if TOPT_ASM_TMA
    if (tma_on) {
      tma::mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int f = 0; f < LPR; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e) z[f][e] = stg[(f * LPB + line) * N + t + T * e];
      __syncthreads();  // every value is in registers: the buffer takes the next group
      if (threadIdx.x == 0 && grp + (int)gridDim.x < ngroups) issue(grp + gridDim.x);
    } else
#endif
    {
#pragma unroll
      for (int f = 0; f < LPR; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e) z[f][e] = ok ? a.Z[f][o + T * e] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int f = 0; f < LPR; ++f) rf_fft<N, E, true, WARP, true>(z[f], lbuf, t, tw);
    if (!ok) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c >= g.d) break;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const size_t gi = (size_t)c * g.F + o + T * e;
        const float2 pz = z[pf + c / 2][e];
        const float pc = (c & 1) ? pz.y : pz.x;
        float bl;
        if constexpr (LERAY) {
          const float2 bz = z[c / 2][e];
          bl = (c & 1) ? bz.y : bz.x;
        } else {
          bl = a.b ? __ldg(a.b + gi) : 0.f;
        }
        const float uc = a.u ? __ldg(a.u + gi) : 0.f;
        const float vc = a.v ? __ldg(a.v + gi) : 0.f;
        const float gv = uc + bl;
        const float sv = vbar[c] - vc + pc;
        if (a.g) a.g[gi] = gv;
        if (a.s) a.s[gi] = sv;
        gmax = fmaxf(gmax, fabsf(gv));
        sgs += (double)(gv * sv);
        svu += (double)vc * uc;
        ssu += (double)sv * uc;
        sg[c] += (double)gv;
        ss[c] += (double)sv;
      }
    }
  }
  double vals[10] = {(double)gmax, sgs, svu, ssu, sg[0], sg[1], sg[2], ss[0], ss[1], ss[2]};
  __shared__ double sh[10][kThreads / 32];
  const int nw = (blockDim.x + 31) / 32;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    double v = vals[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double w = __shfl_down_sync(0xffffffffu, v, off);
      v = k == 0 ? fmax(v, w) : v + w;
    }
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    const int k = threadIdx.x;
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc = k == 0 ? fmax(acc, sh[k][w]) : acc + sh[k][w];
    a.partials[(size_t)k * kMaxPartials + blockIdx.x] = acc;
  }
}

// ---- launchers ------------------------------------------------------------------------
template <int N, int EMAX, typename C>
static void rx_fwd_launch(const Geom& g, const RealIn& in, const ZList<C>& Z, int nf, cudaStream_t st) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E, LPB = kThreads / T;
  const size_t sm = (size_t)LPB * RfCfg<N, E>::STRIDE * sizeof(C);
  const size_t nrows = (size_t)g.ny * g.nz;
  const long long groups = (long long)((nrows + LPB - 1) / LPB);
  const int bx = persistent_blocks(k_rx_fwd<N, EMAX, C>, kThreads, sm, groups * nf);
  const int per = (bx + nf - 1) / nf;
  k_rx_fwd<N, EMAX, C><<<dim3(per, nf), kThreads, sm, st>>>(g, in, Z, (int)groups);
  count_launch();
}

template <int N, int EMAX, typename C>
static void rx_inv_launch(const Geom& g, const ZList<C>& Z, const RealOut& out, int nf, cudaStream_t st) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E, LPB = kThreads / T;
  const size_t sm = (size_t)LPB * RfCfg<N, E>::STRIDE * sizeof(C);
  const size_t nrows = (size_t)g.ny * g.nz;
  const long long groups = (long long)((nrows + LPB - 1) / LPB);
  const int bx = persistent_blocks(k_rx_inv<N, EMAX, C>, kThreads, sm, groups * nf);
  const int per = (bx + nf - 1) / nf;
  k_rx_inv<N, EMAX, C><<<dim3(per, nf), kThreads, sm, st>>>(g, Z, out, (int)groups);
  count_launch();
}

// TMA-staged form of the y / z passes without a spectral operator (k_rstrided MODE 0 forward,
// MODE 1 inverse; one field per work item, in place): the N x TXC complex tile of the next item
// arrives by one TMA tensor copy (3D map of the field, complex as 2 reals) while the current one is
// transformed, into a two-slot ring; the tile doubles as the exchange scratch (interleaved,
// swizzled).  128 threads, 32 KB of tiles: several blocks per SM.
struct TmaZ {
  CUtensorMap m[4];
};
constexpr int kRsThreads = 128;
template <int N, int EMAX, int MODE, typename C>
__global__ void __launch_bounds__(kRsThreads, 3) k_rstrided_tma(Geom g, int axis, const __grid_constant__ TmaZ tm,
                                                                 ZList<C> Z, int nitems) {
  static_assert(MODE == 0 || MODE == 1, "plain forward / inverse passes");
  constexpr int E = Ev<N, EMAX>::v, T = N / E, TXC = kRsThreads / T;
  constexpr int TILE = N * TXC;                // complex per tile
  constexpr int BOX = N < 256 ? N : 256;
  using Tr = typename Real<C>::T;
  extern __shared__ __align__(128) unsigned char smr[];
  C* tiles = reinterpret_cast<C*>(smr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(tiles + 2 * TILE);
  const int c = threadIdx.x % TXC, t = threadIdx.x / TXC;
  C tw[RfCfg<N, E>::NTW];
  rf_twiddles<N, E>(tw, t);
  const int tilesx = g.nx / TXC;
  const int outerN = axis == 1 ? g.nz : g.ny;
  const int tiles_per_field = tilesx * outerN;
  const size_t Su = axis == 1 ? (size_t)g.nx : (size_t)g.nx * g.ny;
  const int nmine = blockIdx.x < nitems ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto issue = [&](int k) {
    const int item = blockIdx.x + k * gridDim.x;
    const int tt = item % tiles_per_field, f = item / tiles_per_field;
    const int x0 = (tt % tilesx) * TXC, outer = tt / tilesx;
    C* dst = tiles + (k & 1) * TILE;
    tma::mbar_arrive_expect_tx(bars + (k & 1), (unsigned)(TILE * sizeof(C)));
    for (int p0 = 0; p0 < N; p0 += BOX)
      tma::tensor4_g2s(dst + p0 * TXC, &tm.m[f], 2 * x0, axis == 1 ? p0 : outer, axis == 1 ? outer : p0, 0,
                       bars + (k & 1));
  };
  if (threadIdx.x == 0) {
    tma::mbar_init(bars, 1);
    tma::mbar_init(bars + 1, 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && nmine > 0) issue(0);
  for (int k = 0; k < nmine; ++k) {
    const int item = blockIdx.x + k * gridDim.x;
    const int tt = item % tiles_per_field, f = item / tiles_per_field;
    const int x0 = (tt % tilesx) * TXC, outer = tt / tilesx;
    TOPT_STRESS_POINT(k * 3 + 61);
    if (threadIdx.x == 0 && k + 1 < nmine) issue(k + 1);
    tma::mbar_wait(bars + (k & 1), (unsigned)(k >> 1) & 1u);
    C* tp = tiles + (k & 1) * TILE;
    C a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = tp[(t + T * e) * TXC + c];
    __syncthreads();  // the tile becomes the exchange scratch
    rf_fft<N, E, MODE == 1, false, false, TXC>(a, tp + c, t, tw);
    C* dstg = Z.z[f] + (axis == 1 ? ((size_t)outer << (g.lx + g.ly)) : ((size_t)outer << g.lx)) + x0 + c;
#pragma unroll
    for (int e = 0; e < E; ++e) dstg[(t + T * e) * Su] = a[e];
    (void)sizeof(Tr);
    TOPT_STRESS_POINT(k * 3 + 62);
    __syncthreads();  // slot k&1 free for item k+2
  }
}

#ifndef TOPT_RS_TMA
#define TOPT_RS_TMA 1
#endif
template <typename C>
static bool field_map(CUtensorMap* m, const C* base, const Geom& g, int axis, int box_x, int box_n) {
  auto enc = tensor_map_encoder();
  if (!enc || (((uintptr_t)base) & 15)) return false;
  // complex as 2 reals: dims (2 nx, ny, nz, 1)
  const CUtensorMapDataType dt = sizeof(C) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const cuuint64_t es = sizeof(C) / 2;
  const cuuint64_t dims[4] = {(cuuint64_t)2 * g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz, 1};
  const cuuint64_t strides[3] = {(cuuint64_t)g.nx * sizeof(C), (cuuint64_t)g.nx * g.ny * sizeof(C),
                                 (cuuint64_t)g.F * sizeof(C)};
  const cuuint32_t box[4] = {(cuuint32_t)(2 * box_x), (cuuint32_t)(axis == 1 ? box_n : 1),
                             (cuuint32_t)(axis == 1 ? 1 : box_n), 1u};
  const cuuint32_t ones[4] = {1, 1, 1, 1};
  (void)es;
  return enc(m, dt, 4, const_cast<C*>(base), dims, strides, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
template <int N, int EMAX, int MODE, typename C>
static bool rstrided_tma_launch(const Geom& g, int axis, const ZList<C>& Z, int nin, cudaStream_t st) {
  if constexpr (MODE > 1) {
    return false;
  } else {
    constexpr int E = Ev<N, EMAX>::v, T = N / E, TXC = kRsThreads / T;
    if (!TOPT_RS_TMA || N < 128 || N > 1024 || TXC < 2 || TXC * (int)sizeof(C) < 16 || g.nx % TXC || nin > 4)
      return false;
    TmaZ tm{};
    for (int f = 0; f < nin; ++f)
      if (!field_map(&tm.m[f], Z.z[f], g, axis, TXC, N < 256 ? N : 256)) return false;
    const size_t sm = 2 * (size_t)N * TXC * sizeof(C) + 2 * sizeof(uint64_t);
    const int outer = axis == 1 ? g.nz : g.ny;
    const long long items = (long long)(g.nx / TXC) * outer * nin;
    const int blocks = persistent_blocks(k_rstrided_tma<N, EMAX, MODE, C>, kRsThreads, sm, items);
    k_rstrided_tma<N, EMAX, MODE, C><<<blocks, kRsThreads, sm, st>>>(g, axis, tm, Z, (int)items);
    count_launch();
    return true;
  }
}

template <int N, int EMAX, int MODE, typename C>
static void rstrided_launch(const Geom& g, int axis, const ZList<C>& Z, int nin, int nout, const SpecOp& op,
                            cudaStream_t st) {
  if (MODE <= 1 && nin == nout && rstrided_tma_launch<N, EMAX, MODE, C>(g, axis, Z, nin, st)) return;
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  int TXC = kThreads / T;
  if (TXC > g.nx) TXC = g.nx;
  const int threads = TXC * T;
  const size_t sm = (size_t)TXC * RfCfg<N, E>::STRIDE * sizeof(C);
  const int outer = axis == 1 ? g.nz : g.ny;
  const long long items = (long long)(g.nx / TXC) * outer * (MODE >= 4 ? 1 : nin);
  const int blocks = persistent_blocks(k_rstrided<N, EMAX, MODE, C>, threads, sm, items);
  k_rstrided<N, EMAX, MODE, C><<<blocks, threads, sm, st>>>(g, axis, TXC, nin, nout, Z, op, (int)items);
  count_launch();
}

template <int N, int EMAX, int MODE, typename C>
static void rstrided_remote_launch(const Geom& gy, const RemoteZ& rz, int nin, const SpecOp& op, cudaStream_t st) {
  constexpr int E = Ev<N, EMAX>::v, T = N / E;
  int TXC = kThreads / T;
  if (TXC > gy.nx) TXC = gy.nx;
  const int threads = TXC * T;
  const size_t sm = (size_t)TXC * RfCfg<N, E>::STRIDE * sizeof(C);
  const long long items = (long long)(gy.nx / TXC) * gy.ny * nin;
  const int blocks = persistent_blocks(k_rstrided<N, EMAX, MODE, C, true>, threads, sm, items);
  ZList<C> Z{};
  k_rstrided<N, EMAX, MODE, C, true><<<blocks, threads, sm, st>>>(gy, 2, TXC, nin, nin, Z, op, (int)items, rz);
  count_launch();
}

#define TOPT_DISPATCH_N2(NV, BODY)                                  \
  switch (NV) {                                                     \
    case 8: { constexpr int N_ = 8; BODY; } break;                  \
    case 16: { constexpr int N_ = 16; BODY; } break;                \
    case 32: { constexpr int N_ = 32; BODY; } break;                \
    case 64: { constexpr int N_ = 64; BODY; } break;                \
    case 128: { constexpr int N_ = 128; BODY; } break;              \
    case 256: { constexpr int N_ = 256; BODY; } break;              \
    case 512: { constexpr int N_ = 512; BODY; } break;              \
    case 1024: { constexpr int N_ = 1024; BODY; } break;            \
    default: fprintf(stderr, "topt: unsupported N %d\n", NV);       \
  }

constexpr int kE32 = 16;  // fp32 single-field lines
constexpr int kE64 = 8;   // fp64 lines and multi-field (Leray) lines

// ---- chain phases (the z pass may run on a y-slab geometry between two transposes) ----------
int vchain_nin(const Geom& g, bool leray) { return leray ? g.d : (g.d == 3 ? 2 : 1); }
int vchain_nout(const Geom& g) { return g.d == 3 ? 2 : 1; }
int bchain_nin(const Geom& g, bool leray) { return leray ? g.d : (g.d == 3 ? 2 : 1); }
int bchain_nout(const Geom& g, bool leray) { return leray ? (g.d == 3 ? 4 : 2) : (g.d == 3 ? 2 : 1); }

void vchain_xy(const Geom& g, const float* v, double2* const* Z, bool leray, cudaStream_t st) {
  const size_t F = g.F;
  ZList<double2> L{{Z[0], Z[1], Z[2], nullptr}};
  RealIn in{};
  const int nin = vchain_nin(g, leray);
  if (leray) {
    for (int c = 0; c < g.d; ++c) { in.re[c] = v + c * F; in.im[c] = nullptr; }
  } else {
    in.re[0] = v; in.im[0] = v + F;
    if (g.d == 3) { in.re[1] = v + 2 * F; in.im[1] = nullptr; }
  }
  SpecOp op{0.0, 1, 1.0};
  TOPT_DISPATCH_N2(g.nx, (rx_fwd_launch<N_, kE64, double2>(g, in, L, nin, st)));
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (rstrided_launch<N_, kE64, 0, double2>(g, 1, L, nin, nin, op, st)));
}

// z pass (3D) or y pass (2D) with the spectral operator, on geometry gz (z-slab when P == 1,
// y-slab [nz][ny/P][nx] with ky0 / nyg set otherwise).  n_total = global point count.
void vchain_last(const Geom& gz, double2* const* Z, double alpha, int p, bool leray, double n_total,
                 cudaStream_t st) {
  ZList<double2> L{{Z[0], Z[1], Z[2], nullptr}};
  SpecOp op{alpha, p, 1.0 / n_total};
  const int nin = vchain_nin(gz, leray), nout = vchain_nout(gz);
  const int axis = gz.d == 3 ? 2 : 1, Nl = gz.d == 3 ? gz.nz : gz.ny;
  if (leray) {
    TOPT_DISPATCH_N2(Nl, (rstrided_launch<N_, kE64, 5, double2>(gz, axis, L, nin, nout, op, st)));
  } else {
    TOPT_DISPATCH_N2(Nl, (rstrided_launch<N_, kE64, 2, double2>(gz, axis, L, nin, nout, op, st)));
  }
}

void vchain_inv(const Geom& g, double2* const* Z, float* u, cudaStream_t st) {
  const size_t F = g.F;
  ZList<double2> L{{Z[0], Z[1], Z[2], nullptr}};
  const int nout = vchain_nout(g);
  SpecOp op{0.0, 1, 1.0};
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (rstrided_launch<N_, kE64, 1, double2>(g, 1, L, nout, nout, op, st)));
  RealOut out{{u, g.d == 3 ? u + 2 * F : nullptr, nullptr}, {u + F, nullptr, nullptr}};
  TOPT_DISPATCH_N2(g.nx, (rx_inv_launch<N_, kE64, double2>(g, L, out, nout, st)));
}

// b-chain: x (and y) forward passes.
void bchain_xy(const Geom& g, const float* b, float2* const* Z, bool leray, cudaStream_t st) {
  const size_t F = g.F;
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  RealIn in{};
  const int nin = bchain_nin(g, leray);
  if (leray) {
    for (int c = 0; c < g.d; ++c) { in.re[c] = b + c * F; in.im[c] = nullptr; }
  } else {
    in.re[0] = b; in.im[0] = b + F;
    if (g.d == 3) { in.re[1] = b + 2 * F; in.im[1] = nullptr; }
  }
  SpecOp op{0.0, 1, 1.0};
  TOPT_DISPATCH_N2(g.nx, (rx_fwd_launch<N_, kE32, float2>(g, in, L, nin, st)));
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (rstrided_launch<N_, kE32, 0, float2>(g, 1, L, nin, nin, op, st)));
}

void bchain_last(const Geom& gz, float2* const* Z, double alpha, int p, bool leray, double n_total,
                 cudaStream_t st) {
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  SpecOp op{alpha, p, 1.0 / n_total};
  const int nin = bchain_nin(gz, leray), nout = bchain_nout(gz, leray);
  const int axis = gz.d == 3 ? 2 : 1, Nl = gz.d == 3 ? gz.nz : gz.ny;
  if (leray) {
    TOPT_DISPATCH_N2(Nl, (rstrided_launch<N_, kE64, 4, float2>(gz, axis, L, nin, nout, op, st)));
  } else {
    TOPT_DISPATCH_N2(Nl, (rstrided_launch<N_, kE32, 3, float2>(gz, axis, L, nin, nout, op, st)));
  }
}

// z-slabs, P2P transport (3D, non-Leray): last-axis passes in place on the distributed slabs.
// tab[f][q] = rank q's field f (z-slab layout), nzl planes per rank of plane_src elements.
static RemoteZ make_rz(const void* const* tab, int nf, int P, int nzl, size_t plane_src) {
  RemoteZ rz{};
  int l = 0;
  while ((1 << l) < nzl) ++l;
  rz.lnzl = l;
  rz.plane_src = (unsigned)plane_src;
  for (int f = 0; f < nf && f < 4; ++f)
    for (int q = 0; q < P && q < 8; ++q) rz.tab[f][q] = tab[f * P + q];
  return rz;
}
void vchain_last_remote(const Geom& gy, const void* const* tab, int P, int nzl, size_t plane_src, double alpha, int p,
                        double n_total, cudaStream_t st) {
  const RemoteZ rz = make_rz(tab, vchain_nin(gy, false), P, nzl, plane_src);
  SpecOp op{alpha, p, 1.0 / n_total};
  TOPT_DISPATCH_N2(gy.nz, (rstrided_remote_launch<N_, kE64, 2, double2>(gy, rz, vchain_nin(gy, false), op, st)));
}
void bchain_last_remote(const Geom& gy, const void* const* tab, int P, int nzl, size_t plane_src, double alpha, int p,
                        double n_total, cudaStream_t st) {
  const RemoteZ rz = make_rz(tab, bchain_nin(gy, false), P, nzl, plane_src);
  SpecOp op{alpha, p, 1.0 / n_total};
  TOPT_DISPATCH_N2(gy.nz, (rstrided_remote_launch<N_, kE32, 3, float2>(gy, rz, bchain_nin(gy, false), op, st)));
}

// Merged last-axis pass (non-Leray): Zv (fp64 v spectra after x, y) and Zb (fp32 b
// spectra after x, y) -> Zb = g^ (fp32), Zb[half + f] = p^; then the y^-1 pass of all four
// (3D) / two (2D) fields, ready for the Leray-layout assembly with u = b = null.
void gchain_last(const Geom& gz, double2* const* Zv, float2* const* Zb, double alpha, int p, double n_total,
                 double* partials, int* nparts, cudaStream_t st) {
  const int half = gz.d == 3 ? 2 : 1;
  ZList<double2> V{{Zv[0], Zv[1], nullptr, nullptr}};
  ZList<float2> B{{Zb[0], Zb[1], nullptr, nullptr}};
  ZList<float2> Pp{{Zb[half], half > 1 ? Zb[half + 1] : nullptr, nullptr, nullptr}};
  SpecOp op{alpha, p, 1.0 / n_total};
  const int axis = gz.d == 3 ? 2 : 1, Nl = gz.d == 3 ? gz.nz : gz.ny;
  TOPT_DISPATCH_N2(Nl, (rzmerge_launch<N_>(gz, axis, V, B, Pp, half, op, partials, nparts, st)));
}
void gchain_yinv(const Geom& g, float2* const* Z, cudaStream_t st) {
  if (g.d != 3) return;
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  SpecOp op{0.0, 1, 1.0};
  TOPT_DISPATCH_N2(g.ny, (rstrided_launch<N_, kE32, 1, float2>(g, 1, L, 4, 4, op, st)));
}

// y^-1 pass of the b-chain (3D); the x^-1 pass is fused into the assembly.
void bchain_yinv(const Geom& g, float2* const* Z, bool leray, cudaStream_t st) {
  if (g.d != 3) return;
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  const int nout = bchain_nout(g, leray);
  SpecOp op{0.0, 1, 1.0};
  TOPT_DISPATCH_N2(g.ny, (rstrided_launch<N_, kE32, 1, float2>(g, 1, L, nout, nout, op, st)));
}

// single-slab compositions
void launch_vchain(const Geom& g, const float* v, double2* Zv, float* u, double alpha, int p, bool leray,
                   cudaStream_t st) {
  double2* Z[3] = {Zv, Zv + g.F, Zv + 2 * g.F};
  vchain_xy(g, v, Z, leray, st);
  vchain_last(g, Z, alpha, p, leray, (double)g.F, st);
  vchain_inv(g, Z, u, st);
}

void launch_bchain(const Geom& g, const float* b, float2* Zb, double alpha, int p, bool leray, cudaStream_t st) {
  float2* Z[4] = {Zb, Zb + g.F, Zb + 2 * g.F, Zb + 3 * g.F};
  bchain_xy(g, b, Z, leray, st);
  bchain_last(g, Z, alpha, p, leray, (double)g.F, st);
  bchain_yinv(g, Z, leray, st);
}

template <int N, int LPR, bool LERAY>
static void rassemble_launch(const Geom& g, const AsmArgs& a, int* nparts, cudaStream_t st) {
  constexpr int E = Ev<N, (LPR >= 4 ? 8 : 16)>::v, T = N / E, LPB = kThreads / T;
  const size_t sm = (size_t)LPB * RfCfg<N, E, true>::STRIDE * sizeof(float2) +
                    (TOPT_ASM_TMA ? (size_t)LPR * LPB * N * sizeof(float2) + sizeof(uint64_t) : 0);
  const size_t nrows = (size_t)g.ny * g.nz;
  const long long groups = (long long)((nrows + LPB - 1) / LPB);
  const int blocks = persistent_blocks(k_rassemble<N, LPR, LERAY>, kThreads, sm, groups);
  *nparts = blocks;
  k_rassemble<N, LPR, LERAY><<<blocks, kThreads, sm, st>>>(g, a, (int)groups);
  count_launch();
}

template <int N>
static void assemble_launch(const Geom& g, bool leray, const AsmArgs& a, int* nparts, cudaStream_t st) {
  const int half = g.d == 3 ? 2 : 1;
  const int lpr = leray ? 2 * half : half;
  if (lpr == 1) rassemble_launch<N, 1, false>(g, a, nparts, st);
  else if (lpr == 2 && leray) rassemble_launch<N, 2, true>(g, a, nparts, st);
  else if (lpr == 2) rassemble_launch<N, 2, false>(g, a, nparts, st);
  else rassemble_launch<N, 4, true>(g, a, nparts, st);
}

void launch_assemble(const Geom& g, const float2* Zb, bool leray, const float* b, const float* u, const float* v,
                     const double* vsum, float* gout, float* sout, double* partials, int* nparts, cudaStream_t st,
                     double ntot) {
  const size_t F = g.F;
  AsmArgs a{{Zb, Zb + F, Zb + 2 * F, Zb + 3 * F}, b, u, v, vsum, gout, sout, partials, ntot > 0 ? ntot : (double)F};
  TOPT_DISPATCH_N(g.nx, assemble_launch, g, leray, a, nparts, st);
}

}  // namespace topt
