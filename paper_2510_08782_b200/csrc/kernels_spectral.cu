// kernels_spectral.cu — pseudo-spectral derivative / body-force kernels and the fused
// 3D-FFT preconditioner (sm_100a).
//
// Fourier pseudo-spectral discretisation, operators applied "at
// the cost of two FFTs and a diagonal scaling"; zero spectral entries of L set to 1
// before inversion.  (2.2) P:105-108 body force int lam grad m dt (trapezoid);
// (2.6) P:172 s = -(alpha L)^{-1} g; incompressible Leray projection (R9).
// Readings: R2 (k range), R3 (Nyquist zeroed for odd derivatives / Leray, true value
// in L), R4 (L = |k|^{2p}), R8 (continuity body force), R23 (reg by Parseval).
//
// Layout of the complex preconditioner buffer Z_c (one per component, F complex):
// after the forward x (and, in 3D, y) passes, spectra are stored in "paired" order
// along those axes so that k and -k sit in the same aligned pair of positions:
//   q = 0 -> 0, q = N/2 -> 1, 0 < q < N/2 -> 2q, N/2 < q < N -> 2(N-q)+1.
// The last axis stays in natural order.  The fused last-axis kernel therefore sees
// every (k, -k) pair inside one tile and can separate Z = v^ + i b^ into v^ and b^.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "fft.cuh"
#include "internal.cuh"

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

template <int N, int RMAX = 16>
struct LineCfg {
  static constexpr int T = fft_threads(N, RMAX);
  static constexpr int LPB = kThreads / T;           // complex lines per 256-thread block
  static constexpr int STRIDE = fft_line_stride(N);  // complex elements per smem line
};

// max radix per element type: fp64 lines use radix 8 (half the registers / smem per thread)
template <typename C> struct RM { static constexpr int v = 16; };
template <> struct RM<double2> { static constexpr int v = 8; };

__device__ __forceinline__ int paired_pos(int q, int N) {  // natural index -> paired position
  return q == 0 ? 0 : (q == N / 2 ? 1 : (q < N / 2 ? 2 * q : 2 * (N - q) + 1));
}
__device__ __forceinline__ int paired_q(int p, int N) {    // paired position -> natural index
  return p == 0 ? 0 : (p == 1 ? N / 2 : ((p & 1) == 0 ? p / 2 : N - (p - 1) / 2));
}
__device__ __forceinline__ float kfreq(int q, int N) { return (float)(q <= N / 2 ? q : q - N); }
__device__ __forceinline__ float kprime(int q, int N) {  // Nyquist zeroed (R3)
  return q == N / 2 ? 0.0f : kfreq(q, N);
}

// =====================================================================================
// Derivative / body-force accumulation along x (contiguous lines).  Two real lines are
// packed into one complex line; the odd multiplier i k' maps real to real (R3), so
// IFFT(i k' FFT(a + i b)) = d a + i d b.
// =====================================================================================
template <int N>
__global__ void __launch_bounds__(kThreads, 3) k_deriv_x(Geom g, const float* __restrict__ psi,
                                                      size_t psi_stride, const float* __restrict__ lam,
                                                      size_t lam_stride, DerivWeights w, int J,
                                                      float beta, float* __restrict__ out) {
  using C = LineCfg<N, 8>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  constexpr int REG4 = (2 * C::LPB * N / 4) / kThreads;  // float4 per thread in the region
  const size_t nlines = (size_t)g.ny * g.nz;               // real lines
  const size_t line0 = (size_t)blockIdx.x * 2 * C::LPB;
  const size_t region0 = line0 * N;                        // first float of the region
  const size_t regionEnd = nlines * N;
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  const bool active = myline < C::LPB;
  float4 acc[REG4];
#pragma unroll
  for (int e = 0; e < REG4; ++e) acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float invN = 1.0f / (float)N;
  for (int j = 0; j < J; ++j) {
    const float* src = psi + j * psi_stride;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < REG4; ++e) {
      const int f4 = threadIdx.x + e * kThreads;  // float4 index within region
      const size_t gi = region0 + (size_t)f4 * 4;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gi < regionEnd) val = *reinterpret_cast<const float4*>(src + gi);
      const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
      float* base = reinterpret_cast<float*>(buf + (rl >> 1) * C::STRIDE) + (rl & 1);
      base[2 * fft_pad(pos + 0)] = val.x;
      base[2 * fft_pad(pos + 1)] = val.y;
      base[2 * fft_pad(pos + 2)] = val.z;
      base[2 * fft_pad(pos + 3)] = val.w;
    }
    __syncthreads();
    float2* line = buf + myline * C::STRIDE;
    fft_line<N, false, 8>(line, tw, tid, active);
    if (active) {
      for (int q = tid; q < N; q += C::T) {
        const float k = kprime(q, N) * invN;
        const float2 z = line[fft_pad(q)];
        line[fft_pad(q)] = make_float2(-k * z.y, k * z.x);  // i k' z / N
      }
    }
    __syncthreads();
    fft_line<N, true, 8>(line, tw, tid, active);
    const float wj = w.w[j];
    const float* lj = lam ? lam + j * lam_stride : nullptr;
#pragma unroll
    for (int e = 0; e < REG4; ++e) {
      const int f4 = threadIdx.x + e * kThreads;
      const size_t gi = region0 + (size_t)f4 * 4;
      const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
      const float* base = reinterpret_cast<const float*>(buf + (rl >> 1) * C::STRIDE) + (rl & 1);
      float4 l4 = make_float4(1.f, 1.f, 1.f, 1.f);
      if (lj && gi < regionEnd) l4 = *reinterpret_cast<const float4*>(lj + gi);
      acc[e].x = fmaf(wj * l4.x, base[2 * fft_pad(pos + 0)], acc[e].x);
      acc[e].y = fmaf(wj * l4.y, base[2 * fft_pad(pos + 1)], acc[e].y);
      acc[e].z = fmaf(wj * l4.z, base[2 * fft_pad(pos + 2)], acc[e].z);
      acc[e].w = fmaf(wj * l4.w, base[2 * fft_pad(pos + 3)], acc[e].w);
    }
  }
#pragma unroll
  for (int e = 0; e < REG4; ++e) {
    const int f4 = threadIdx.x + e * kThreads;
    const size_t gi = region0 + (size_t)f4 * 4;
    if (gi >= regionEnd) continue;
    float4* o = reinterpret_cast<float4*>(out + gi);
    float4 r = acc[e];
    if (beta != 0.0f) {
      const float4 p = *o;
      r.x += beta * p.x; r.y += beta * p.y; r.z += beta * p.z; r.w += beta * p.w;
    }
    *o = r;
  }
}

// =====================================================================================
// Derivative / body-force accumulation along a strided axis (y or z).  A block owns a
// tile of TX consecutive x columns x N positions; columns (2c, 2c+1) share a complex line.
// =====================================================================================
template <int N>
__global__ void __launch_bounds__(kThreads, 3) k_deriv_strided(Geom g, int axis, int TX,
                                                               const float* __restrict__ psi,
                                                               size_t psi_stride,
                                                               const float* __restrict__ lam,
                                                               size_t lam_stride, DerivWeights w, int J,
                                                               float beta, float* __restrict__ out) {
  using C = LineCfg<N, 8>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  // all threads active: threads = (TX/2) * T, float4 per thread = N / (2T) = E4
  constexpr int E4 = N / (2 * C::T);
  const int TX4 = TX >> 2;
  const int lt4 = __ffs(TX4) - 1;
  const int tilesx = g.nx / TX;
  const int x0 = (blockIdx.x % tilesx) * TX;
  const int outer = blockIdx.x / tilesx;
  unsigned base, S;
  if (axis == 1) { base = ((unsigned)outer << (g.lx + g.ly)) + x0; S = g.nx; }
  else { base = ((unsigned)outer << g.lx) + x0; S = (unsigned)g.nx * g.ny; }
  unsigned goff[E4];
  int soff[E4];
#pragma unroll
  for (int e = 0; e < E4; ++e) {
    const int f4 = threadIdx.x + e * blockDim.x;
    const int row = f4 >> lt4, c4 = f4 & (TX4 - 1);
    goff[e] = base + row * S + 4 * c4;
    soff[e] = (2 * c4) * C::STRIDE + fft_pad(row);
  }
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  float4 acc[E4];
#pragma unroll
  for (int e = 0; e < E4; ++e) acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float invN = 1.0f / (float)N;
  for (int j = 0; j < J; ++j) {
    const float* src = psi + j * psi_stride;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E4; ++e) {
      const float4 val = __ldg(reinterpret_cast<const float4*>(src + goff[e]));
      buf[soff[e]] = make_float2(val.x, val.y);
      buf[soff[e] + C::STRIDE] = make_float2(val.z, val.w);
    }
    __syncthreads();
    float2* line = buf + myline * C::STRIDE;
    fft_line<N, false, 8>(line, tw, tid, true);
    for (int q = tid; q < N; q += C::T) {
      const float k = kprime(q, N) * invN;
      const float2 z = line[fft_pad(q)];
      line[fft_pad(q)] = make_float2(-k * z.y, k * z.x);
    }
    __syncthreads();
    fft_line<N, true, 8>(line, tw, tid, true);
    const float wj = w.w[j];
    const float* lj = lam ? lam + j * lam_stride : nullptr;
#pragma unroll
    for (int e = 0; e < E4; ++e) {
      const float2 d0 = buf[soff[e]];
      const float2 d1 = buf[soff[e] + C::STRIDE];
      float4 l4 = make_float4(1.f, 1.f, 1.f, 1.f);
      if (lj) l4 = __ldg(reinterpret_cast<const float4*>(lj + goff[e]));
      acc[e].x = fmaf(wj * l4.x, d0.x, acc[e].x);
      acc[e].y = fmaf(wj * l4.y, d0.y, acc[e].y);
      acc[e].z = fmaf(wj * l4.z, d1.x, acc[e].z);
      acc[e].w = fmaf(wj * l4.w, d1.y, acc[e].w);
    }
  }
#pragma unroll
  for (int e = 0; e < E4; ++e) {
    float4* o = reinterpret_cast<float4*>(out + goff[e]);
    float4 r = acc[e];
    if (beta != 0.0f) {
      const float4 p = *o;
      r.x += beta * p.x; r.y += beta * p.y; r.z += beta * p.z; r.w += beta * p.w;
    }
    *o = r;
  }
}

template <int N, int RMAX = 16>
static size_t line_smem() {
  using C = LineCfg<N, RMAX>;
  return (size_t)(C::LPB * C::STRIDE + N) * sizeof(float2);
}

template <int N>
static void deriv_dispatch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w,
                           cudaStream_t st) {
  using C = LineCfg<N, 8>;
  const size_t sm = line_smem<N, 8>();
  if (axis == 0) {
    const size_t nlines = (size_t)g.ny * g.nz;
    const int blocks = (int)((nlines + 2 * C::LPB - 1) / (2 * C::LPB));
    cudaFuncSetAttribute(k_deriv_x<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_deriv_x<N><<<blocks, kThreads, sm, st>>>(g, a.psi, a.psi_stride, a.lam, a.lam_stride, w, a.J,
                                                a.beta, a.out);
  } else {
    int TX = 2 * C::LPB;
    if (TX > g.nx) TX = g.nx;
    const int outer = axis == 1 ? g.nz : g.ny;
    const int blocks = (g.nx / TX) * outer;
    const int threads = (TX / 2) * C::T;
    cudaFuncSetAttribute(k_deriv_strided<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_deriv_strided<N><<<blocks, threads, sm, st>>>(g, axis, TX, a.psi, a.psi_stride, a.lam,
                                                     a.lam_stride, w, a.J, a.beta, a.out);
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

void launch_deriv_accum(const Geom& g, int axis, const DerivArgs& a, cudaStream_t st) {
  DerivWeights w;
  for (int j = 0; j < a.J && j < kMaxWeights; ++j) w.w[j] = (float)a.w[j];
  const int N = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  TOPT_DISPATCH_N(N, deriv_dispatch, g, axis, a, w, st);
}

// =====================================================================================
// Preconditioner / regulariser chains (3D FFT = x pass, [y pass], last-axis pass with a
// fused spectral operator, [y^-1], x^-1).  Spectra stay in natural order.
//
//  v-chain (fp64 arithmetic AND fp64 intermediates): u = alpha L v.  L = |k|^{2p}
//    amplifies any rounding at high |k| by up to (k_max/k)^{2p}, so the chain that
//    applies it runs in double; packing v_x + i v_y is exact because
//    alpha L(k) is real and even.
//  b-chain (fp32): the smoothing inverse -(alpha L~)^{-1} and the Leray projector are
//    well conditioned.  Non-Leray: Z0 = b_x + i b_y, Z1 = b_z -> W = -Z/(alpha L~ n) gives
//    p = -(alpha L~)^{-1} b.  Leray (R3, R9): Z_c = b_c (real, c < d); at each k the
//    projected b_L^ = P_L b^ and p^ = -b_L^/(alpha L~) are written as separate pairs
//    (b_Lx + i b_Ly), (b_Lz), (p_x + i p_y), (p_z) — never b_L and p in one complex field,
//    whose magnitudes differ by up to 1/alpha and would pollute each other in fp32.
//  Incompressible v-chain: Z_c = v_c (fp64) -> (u_x + i u_y), (u_z), u = alpha L P_L v.
// =====================================================================================
template <typename C>
struct ZList { C* z[4]; };
struct RealIn { const float* re[3]; const float* im[3]; };

// x pass forward: Z_f[row][q] = FFT_x(re_f + i im_f)[q]
template <int N, typename C>
__global__ void __launch_bounds__(kThreads) k_px_fwd(Geom g, RealIn in, ZList<C> Z) {
  using L = LineCfg<N, RM<C>::v>;
  using T = typename Real<C>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* buf = reinterpret_cast<C*>(smraw);
  C* tw = buf + L::LPB * L::STRIDE;
  load_twiddles<N>(tw);
  const size_t nrows = (size_t)g.ny * g.nz;
  const size_t row0 = (size_t)blockIdx.x * L::LPB;
  const int f = blockIdx.y;
  const float* re = in.re[f];
  const float* im = in.im[f];
  C* Zf = Z.z[f];
  const int n4 = L::LPB * N / 4;
  for (int f4 = threadIdx.x; f4 < n4; f4 += kThreads) {
    const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
    const size_t gi = (row0 + rl) * N + pos;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (row0 + rl < nrows) {
      if (re) a = *reinterpret_cast<const float4*>(re + gi);
      if (im) b = *reinterpret_cast<const float4*>(im + gi);
    }
    C* Ln = buf + rl * L::STRIDE;
    Ln[fft_pad(pos + 0)] = mk((T)a.x, (T)b.x);
    Ln[fft_pad(pos + 1)] = mk((T)a.y, (T)b.y);
    Ln[fft_pad(pos + 2)] = mk((T)a.z, (T)b.z);
    Ln[fft_pad(pos + 3)] = mk((T)a.w, (T)b.w);
  }
  __syncthreads();
  const int myline = threadIdx.x / L::T, tid = threadIdx.x % L::T;
  fft_line<N, false, RM<C>::v>(buf + myline * L::STRIDE, tw, tid, myline < L::LPB);
  for (int i = threadIdx.x; i < L::LPB * N; i += kThreads) {
    const int rl = i / N, q = i % N;
    if (row0 + rl < nrows) Zf[(row0 + rl) * N + q] = buf[rl * L::STRIDE + fft_pad(q)];
  }
}

// x pass inverse to real outputs: re_f + i im_f = IFFT_x(Z_f)  (either output may be null)
struct RealOut { float* re[3]; float* im[3]; };
template <int N, typename C>
__global__ void __launch_bounds__(kThreads) k_px_inv(Geom g, ZList<C> Z, RealOut out) {
  using L = LineCfg<N, RM<C>::v>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* buf = reinterpret_cast<C*>(smraw);
  C* tw = buf + L::LPB * L::STRIDE;
  load_twiddles<N>(tw);
  const size_t nrows = (size_t)g.ny * g.nz;
  const size_t row0 = (size_t)blockIdx.x * L::LPB;
  const int f = blockIdx.y;
  const C* Zf = Z.z[f];
  for (int i = threadIdx.x; i < L::LPB * N; i += kThreads) {
    const int rl = i / N, q = i % N;
    C z = mk((typename Real<C>::T)0, (typename Real<C>::T)0);
    if (row0 + rl < nrows) z = Zf[(row0 + rl) * N + q];
    buf[rl * L::STRIDE + fft_pad(q)] = z;
  }
  __syncthreads();
  const int myline = threadIdx.x / L::T, tid = threadIdx.x % L::T;
  fft_line<N, true, RM<C>::v>(buf + myline * L::STRIDE, tw, tid, myline < L::LPB);
  float* re = out.re[f];
  float* im = out.im[f];
  const int n4 = L::LPB * N / 4;
  for (int f4 = threadIdx.x; f4 < n4; f4 += kThreads) {
    const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
    if (row0 + rl >= nrows) continue;
    const size_t gi = (row0 + rl) * N + pos;
    const C* Ln = buf + rl * L::STRIDE;
    const C a0 = Ln[fft_pad(pos)], a1 = Ln[fft_pad(pos + 1)], a2 = Ln[fft_pad(pos + 2)], a3 = Ln[fft_pad(pos + 3)];
    if (re) *reinterpret_cast<float4*>(re + gi) = make_float4((float)a0.x, (float)a1.x, (float)a2.x, (float)a3.x);
    if (im) *reinterpret_cast<float4*>(im + gi) = make_float4((float)a0.y, (float)a1.y, (float)a2.y, (float)a3.y);
  }
}

// Strided-axis pass (lines along y in 3D, along the last axis otherwise).  A tile is TXC
// consecutive complex columns of NIN fields (Leray modes: the d components together),
// written back as NOUT fields.
//   MODE 0: forward FFT only        (3D y pass)
//   MODE 1: inverse FFT only        (3D y^-1 pass)
//   MODE 2: fwd, Z *= alpha L(k)/n, inv                        (v-chain, last axis)
//   MODE 3: fwd, Z *= -1/(alpha L~(k) n), inv                  (b-chain, last axis)
//   MODE 4: fwd, Leray + inverse regulariser, inv; d -> 2 (2D) / 4 (3D) fields (b-chain)
//   MODE 5: fwd, alpha L P_L, inv; d -> 1 (2D) / 2 (3D) fields (incompressible v-chain)
struct SpecOp {
  double alpha;
  int p;
  double invn;
};

__device__ __forceinline__ double regL(double kk, int p) { return p == 1 ? kk : (p == 2 ? kk * kk : kk * kk * kk); }

// cp.async (LDGSTS) helpers: global -> shared copies that bypass registers
__device__ __forceinline__ void cp_async(void* smem, const float2* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_async(void* smem, const double2* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Persistent and double-buffered: a block walks work items (tile x field); the tile of
// item k+1 is copied global -> shared with cp.async while item k is transformed, so HBM
// latency overlaps the FFT instead of stalling every block at a barrier.
template <int N, int MODE, typename C>
__global__ void __launch_bounds__(kThreads) k_pstrided(Geom g, int axis, int TXC, int NIN, int NOUT, ZList<C> Z,
                                                       SpecOp op, int nitems) {
  using L = LineCfg<N, RM<C>::v>;
  using T = typename Real<C>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int NL = NIN > NOUT ? NIN : NOUT;  // line slots per column
  const int lines = NL * TXC;
  C* buf0 = reinterpret_cast<C*>(smraw);
  C* buf1 = buf0 + lines * L::STRIDE;
  C* tw = buf1 + lines * L::STRIDE;
  load_twiddles<N>(tw);
  const int tilesx = g.nx / TXC;
  const int outerN = axis == 1 ? g.nz : g.ny;
  const int tiles = tilesx * outerN;
  const int ltx = __ffs(TXC) - 1;  // TXC is a power of two
  const unsigned Su = axis == 1 ? (unsigned)g.nx : (unsigned)g.nx * g.ny;
  const int nin = NIN * TXC, nout = NOUT * TXC;
  const int myline = threadIdx.x / L::T, tid = threadIdx.x % L::T;

  auto item_geom = [&](int item, int& f0, int& x0, int& outer, unsigned& base) {
    const int t = item % tiles;
    f0 = (MODE >= 4) ? 0 : item / tiles;
    x0 = (t % tilesx) * TXC;
    outer = t / tilesx;
    base = axis == 1 ? ((unsigned)outer << (g.lx + g.ly)) + x0 : ((unsigned)outer << g.lx) + x0;
  };
  auto prefetch = [&](int item, C* buf) {
    int f0, x0, outer;
    unsigned base;
    item_geom(item, f0, x0, outer, base);
    for (int f = 0; f < NIN; ++f) {
      const C* __restrict__ src = Z.z[f0 + f];
      C* dst = buf + f * TXC * L::STRIDE;
      for (int i = threadIdx.x; i < N * TXC; i += blockDim.x) {
        const int row = i >> ltx, c = i & (TXC - 1);
        cp_async(dst + c * L::STRIDE + fft_pad(row), src + base + row * Su + c);
      }
    }
  };

  int item = blockIdx.x;
  bool cur0 = true;
  if (item < nitems) prefetch(item, buf0);
  cp_commit();
  for (; item < nitems; item += gridDim.x, cur0 = !cur0) {
    C* buf = cur0 ? buf0 : buf1;
    const int next = item + gridDim.x;
    if (next < nitems) prefetch(next, cur0 ? buf1 : buf0);
    cp_commit();
    cp_wait_1();  // this item's copies have landed (the next item's may still be in flight)
    __syncthreads();
    int f0, x0, outer;
    unsigned base;
    item_geom(item, f0, x0, outer, base);
    if (MODE != 1) fft_line<N, false, RM<C>::v>(buf + myline * L::STRIDE, tw, tid, myline < nin);
    if (MODE >= 2) {
      for (int i = threadIdx.x; i < N * TXC; i += blockDim.x) {
        const int q = i >> ltx, c = i & (TXC - 1);
        const int qx = x0 + c;
        const double kx = qx <= g.nx / 2 ? qx : qx - g.nx, kxp = qx == g.nx / 2 ? 0.0 : kx;
        double ky, kyp, kz, kzp;
        if (g.d == 3) {
          const int nyg = g.nyg ? g.nyg : g.ny;  // y-slab layout: global row = ky0 + local row
          const int qy = outer + g.ky0;
          ky = qy <= nyg / 2 ? qy : qy - nyg; kyp = qy == nyg / 2 ? 0.0 : ky;
          kz = q <= N / 2 ? q : q - N; kzp = q == N / 2 ? 0.0 : kz;
        } else {
          ky = q <= N / 2 ? q : q - N; kyp = q == N / 2 ? 0.0 : ky;
          kz = 0.0; kzp = 0.0;
        }
        const double Lk = regL(kx * kx + ky * ky + kz * kz, op.p);
        const double Lt = Lk == 0.0 ? 1.0 : Lk;  // kernel fix
        if (MODE == 2 || MODE == 3) {
          // the smoothing multiplier in float (relative 1e-7); no fp64 division
          const T m = MODE == 2 ? (T)(op.alpha * Lk * op.invn)
                                : (T)(-(float)op.invn * __frcp_rn((float)(op.alpha * Lt)));
          C& z = buf[c * L::STRIDE + fft_pad(q)];
          z = mk(z.x * m, z.y * m);
        } else {
          // Leray on the d components at this k (Nyquist-zeroed k', R3/R9)
          const double kp2 = kxp * kxp + kyp * kyp + kzp * kzp;
          const double kp[3] = {kxp, kyp, kzp};
          double bx[3] = {0, 0, 0}, by[3] = {0, 0, 0};
          for (int f = 0; f < NIN; ++f) {
            const C z = buf[(f * TXC + c) * L::STRIDE + fft_pad(q)];
            bx[f] = z.x; by[f] = z.y;
          }
          if (kp2 > 0.0) {
            // per-mode relative precision suffices (a 0-order projector): fp32 reciprocal
            const double ikp = (double)__frcp_rn((float)kp2);
            double dx = 0.0, dy = 0.0;
            for (int f = 0; f < NIN; ++f) { dx += kp[f] * bx[f]; dy += kp[f] * by[f]; }
            dx *= ikp;
            dy *= ikp;
            for (int f = 0; f < NIN; ++f) { bx[f] -= kp[f] * dx; by[f] -= kp[f] * dy; }
          }
          // each component's spectrum is bx + i by; pack pairs of REAL fields: A + i B has
          // spectrum A^ + i B^ = (Ax - By) + i (Ay + Bx)
          const double sl = MODE == 5 ? op.alpha * Lk * op.invn : op.invn;
          const double sp = -op.invn * (double)__frcp_rn((float)(op.alpha * Lt));
          auto put = [&](int slot, int a, int b, double sa, double sb) {
            const double ax = a >= 0 ? sa * bx[a] : 0.0, ay = a >= 0 ? sa * by[a] : 0.0;
            const double cx = b >= 0 ? sb * bx[b] : 0.0, cy = b >= 0 ? sb * by[b] : 0.0;
            buf[(slot * TXC + c) * L::STRIDE + fft_pad(q)] = mk((T)(ax - cy), (T)(ay + cx));
          };
          if (g.d == 3) {
            put(0, 0, 1, sl, sl);
            put(1, 2, -1, sl, 0.0);
            if (MODE == 4) { put(2, 0, 1, sp, sp); put(3, 2, -1, sp, 0.0); }
          } else {
            put(0, 0, 1, sl, sl);
            if (MODE == 4) put(1, 0, 1, sp, sp);
          }
        }
      }
      __syncthreads();
    }
    if (MODE != 0) fft_line<N, true, RM<C>::v>(buf + myline * L::STRIDE, tw, tid, myline < nout);
    for (int f = 0; f < NOUT; ++f) {
      C* __restrict__ dst = Z.z[f0 + f];
      const C* src = buf + f * TXC * L::STRIDE;
      for (int i = threadIdx.x; i < N * TXC; i += blockDim.x) {
        const int row = i >> ltx, c = i & (TXC - 1);
        dst[base + row * Su + c] = src[c * L::STRIDE + fft_pad(row)];
      }
    }
    __syncthreads();  // this buffer is refilled by the prefetch issued at the next iteration
  }
  cp_wait_0();
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

template <int N>
__global__ void __launch_bounds__(kThreads) k_assemble(Geom g, int RB, int lpr, int leray, AsmArgs a) {
  using L = LineCfg<N>;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* buf = reinterpret_cast<float2*>(smraw);
  float2* tw = buf + RB * lpr * L::STRIDE;
  load_twiddles<N>(tw);
  const size_t nrows = (size_t)g.ny * g.nz;
  const size_t row0 = (size_t)blockIdx.x * RB;
  const int nlines = RB * lpr;
  for (int i = threadIdx.x; i < nlines * N; i += blockDim.x) {
    const int l = i / N, q = i % N;
    const int r = l >> (lpr >> 1), f = l & (lpr - 1);  // lpr in {1, 2, 4}
    float2 z = make_float2(0.f, 0.f);
    if (row0 + r < nrows) z = a.Z[f][(row0 + r) * N + q];
    buf[l * L::STRIDE + fft_pad(q)] = z;
  }
  __syncthreads();
  const int myline = threadIdx.x / L::T, tid = threadIdx.x % L::T;
  fft_line<N, true>(buf + myline * L::STRIDE, tw, tid, myline < nlines);
  double gmax = 0.0, sgs = 0.0, svu = 0.0, ssu = 0.0, sg[3] = {0, 0, 0}, ss[3] = {0, 0, 0};
  const double nF = a.ntot;
  const int pf = leray ? lpr / 2 : 0;  // first p field
  for (int i4 = threadIdx.x; i4 < RB * N / 4; i4 += blockDim.x) {
    const int r = (4 * i4) / N, x = (4 * i4) % N;
    if (row0 + r >= nrows) continue;
    const size_t gi = (row0 + r) * N + x;
    for (int c = 0; c < g.d; ++c) {
      const size_t o = c * g.F + gi;
      float4 bl, pc;
      {
        const float2* L = buf + (r * lpr + pf + c / 2) * L::STRIDE;
        const float2 w0 = L[fft_pad(x)], w1 = L[fft_pad(x + 1)], w2 = L[fft_pad(x + 2)], w3 = L[fft_pad(x + 3)];
        pc = (c & 1) ? make_float4(w0.y, w1.y, w2.y, w3.y) : make_float4(w0.x, w1.x, w2.x, w3.x);
      }
      if (leray) {
        const float2* L = buf + (r * lpr + c / 2) * L::STRIDE;
        const float2 w0 = L[fft_pad(x)], w1 = L[fft_pad(x + 1)], w2 = L[fft_pad(x + 2)], w3 = L[fft_pad(x + 3)];
        bl = (c & 1) ? make_float4(w0.y, w1.y, w2.y, w3.y) : make_float4(w0.x, w1.x, w2.x, w3.x);
      } else {
        bl = a.b ? __ldg(reinterpret_cast<const float4*>(a.b + o)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const float4 uc = a.u ? __ldg(reinterpret_cast<const float4*>(a.u + o)) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 vc = a.v ? __ldg(reinterpret_cast<const float4*>(a.v + o)) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float vbar = a.vsum ? (float)(a.vsum[c] / nF) : 0.f;
      const float4 gv = make_float4(uc.x + bl.x, uc.y + bl.y, uc.z + bl.z, uc.w + bl.w);
      const float4 sv = make_float4(vbar - vc.x + pc.x, vbar - vc.y + pc.y, vbar - vc.z + pc.z, vbar - vc.w + pc.w);
      if (a.g) *reinterpret_cast<float4*>(a.g + o) = gv;
      if (a.s) *reinterpret_cast<float4*>(a.s + o) = sv;
      gmax = fmax(gmax, (double)fmaxf(fmaxf(fabsf(gv.x), fabsf(gv.y)), fmaxf(fabsf(gv.z), fabsf(gv.w))));
      sgs += (double)(gv.x * sv.x) + (double)(gv.y * sv.y) + (double)(gv.z * sv.z) + (double)(gv.w * sv.w);
      svu += (double)vc.x * uc.x + (double)vc.y * uc.y + (double)vc.z * uc.z + (double)vc.w * uc.w;
      ssu += (double)sv.x * uc.x + (double)sv.y * uc.y + (double)sv.z * uc.z + (double)sv.w * uc.w;
      sg[c] += (double)gv.x + (double)gv.y + (double)gv.z + (double)gv.w;
      ss[c] += (double)sv.x + (double)sv.y + (double)sv.z + (double)sv.w;
    }
  }
  double vals[10] = {gmax, sgs, svu, ssu, sg[0], sg[1], sg[2], ss[0], ss[1], ss[2]};
  __shared__ double sh[10][kThreads / 32];
  const int nw = (blockDim.x + 31) / 32;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    double v = vals[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_down_sync(0xffffffffu, v, o);
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

template <int N, typename C>
static size_t smem_lines(int nlines) {
  return (size_t)(nlines * LineCfg<N, RM<C>::v>::STRIDE + N) * sizeof(C);
}

template <int N, typename C>
static void px_fwd_launch(const Geom& g, const RealIn& in, const ZList<C>& Z, int nf, cudaStream_t st) {
  using L = LineCfg<N, RM<C>::v>;
  const size_t sm = smem_lines<N, C>(L::LPB);
  const size_t nrows = (size_t)g.ny * g.nz;
  dim3 grid((unsigned)((nrows + L::LPB - 1) / L::LPB), nf);
  cudaFuncSetAttribute(k_px_fwd<N, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_px_fwd<N, C><<<grid, kThreads, sm, st>>>(g, in, Z);
  count_launch();
}

template <int N, typename C>
static void px_inv_launch(const Geom& g, const ZList<C>& Z, const RealOut& out, int nf, cudaStream_t st) {
  using L = LineCfg<N, RM<C>::v>;
  const size_t sm = smem_lines<N, C>(L::LPB);
  const size_t nrows = (size_t)g.ny * g.nz;
  dim3 grid((unsigned)((nrows + L::LPB - 1) / L::LPB), nf);
  cudaFuncSetAttribute(k_px_inv<N, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_px_inv<N, C><<<grid, kThreads, sm, st>>>(g, Z, out);
  count_launch();
}

template <int N, int MODE, typename C>
static void pstrided_launch(const Geom& g, int axis, const ZList<C>& Z, int nin, int nout, const SpecOp& op,
                            cudaStream_t st) {
  using L = LineCfg<N, RM<C>::v>;
  const bool multi = MODE >= 4;
  const int NIN = multi ? nin : 1, NOUT = multi ? nout : 1;
  const int NL = NIN > NOUT ? NIN : NOUT;
  int TXC = L::LPB / NL;
  int t = 1;
  while (t * 2 <= TXC) t *= 2;
  TXC = t;
  if (TXC > g.nx) TXC = g.nx;
  if (TXC < 1) TXC = 1;
  const size_t sm = (size_t)(2 * NL * TXC * L::STRIDE + N) * sizeof(C);
  const int outer = axis == 1 ? g.nz : g.ny;
  const int items = (g.nx / TXC) * outer * (multi ? 1 : nin);
  const int threads = NL * TXC * L::T;
  cudaFuncSetAttribute(k_pstrided<N, MODE, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pstrided<N, MODE, C>, threads, sm);
  if (per_sm < 1) per_sm = 1;
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int blocks = nsm * per_sm;
  if (blocks > items) blocks = items;
  k_pstrided<N, MODE, C><<<blocks, threads, sm, st>>>(g, axis, TXC, NIN, NOUT, Z, op, items);
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

// ---- chain phases (the z pass may run on a y-slab geometry between two transposes) ----------
// v-chain: u = alpha L v (P_L first if leray), fp64 arithmetic and intermediates.
// Fields: leray ? d real inputs (v_c + i 0) : (v_x + i v_y)[, (v_z)]; outputs (u_x + i u_y)[, (u_z)].
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
  TOPT_DISPATCH_N2(g.nx, (px_fwd_launch<N_, double2>(g, in, L, nin, st)));
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (pstrided_launch<N_, 0, double2>(g, 1, L, nin, nin, op, st)));
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
    TOPT_DISPATCH_N2(Nl, (pstrided_launch<N_, 5, double2>(gz, axis, L, nin, nout, op, st)));
  } else {
    TOPT_DISPATCH_N2(Nl, (pstrided_launch<N_, 2, double2>(gz, axis, L, nin, nout, op, st)));
  }
}

void vchain_inv(const Geom& g, double2* const* Z, float* u, cudaStream_t st) {
  const size_t F = g.F;
  ZList<double2> L{{Z[0], Z[1], Z[2], nullptr}};
  const int nout = vchain_nout(g);
  SpecOp op{0.0, 1, 1.0};
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (pstrided_launch<N_, 1, double2>(g, 1, L, nout, nout, op, st)));
  RealOut out{{u, g.d == 3 ? u + 2 * F : nullptr, nullptr}, {u + F, nullptr, nullptr}};
  TOPT_DISPATCH_N2(g.nx, (px_inv_launch<N_, double2>(g, L, out, nout, st)));
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
  TOPT_DISPATCH_N2(g.nx, (px_fwd_launch<N_, float2>(g, in, L, nin, st)));
  if (g.d == 3) TOPT_DISPATCH_N2(g.ny, (pstrided_launch<N_, 0, float2>(g, 1, L, nin, nin, op, st)));
}

void bchain_last(const Geom& gz, float2* const* Z, double alpha, int p, bool leray, double n_total,
                 cudaStream_t st) {
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  SpecOp op{alpha, p, 1.0 / n_total};
  const int nin = bchain_nin(gz, leray), nout = bchain_nout(gz, leray);
  const int axis = gz.d == 3 ? 2 : 1, Nl = gz.d == 3 ? gz.nz : gz.ny;
  if (leray) {
    TOPT_DISPATCH_N2(Nl, (pstrided_launch<N_, 4, float2>(gz, axis, L, nin, nout, op, st)));
  } else {
    TOPT_DISPATCH_N2(Nl, (pstrided_launch<N_, 3, float2>(gz, axis, L, nin, nout, op, st)));
  }
}

// y^-1 pass of the b-chain (3D); the x^-1 pass is fused into the assembly.
void bchain_yinv(const Geom& g, float2* const* Z, bool leray, cudaStream_t st) {
  if (g.d != 3) return;
  ZList<float2> L{{Z[0], Z[1], Z[2], Z[3]}};
  const int nout = bchain_nout(g, leray);
  SpecOp op{0.0, 1, 1.0};
  TOPT_DISPATCH_N2(g.ny, (pstrided_launch<N_, 1, float2>(g, 1, L, nout, nout, op, st)));
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

template <int N>
static void assemble_launch(const Geom& g, bool leray, const AsmArgs& a, int* nparts, cudaStream_t st) {
  using L = LineCfg<N>;
  const int half = g.d == 3 ? 2 : 1;
  const int lpr = leray ? 2 * half : half;
  int RB = L::LPB / lpr;
  if (RB < 1) RB = 1;
  const size_t sm = smem_lines<N, float2>(RB * lpr);
  const size_t nrows = (size_t)g.ny * g.nz;
  const int blocks = (int)((nrows + RB - 1) / RB);
  *nparts = blocks;
  cudaFuncSetAttribute(k_assemble<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_assemble<N><<<blocks, RB * lpr * L::T, sm, st>>>(g, RB, lpr, leray ? 1 : 0, a);
  count_launch();
}

void launch_assemble(const Geom& g, const float2* Zb, bool leray, const float* b, const float* u, const float* v,
                     const double* vsum, float* gout, float* sout, double* partials, int* nparts, cudaStream_t st,
                     double ntot) {
  const size_t F = g.F;
  AsmArgs a{{Zb, Zb + F, Zb + 2 * F, Zb + 3 * F}, b, u, v, vsum, gout, sout, partials, ntot > 0 ? ntot : (double)F};
  TOPT_DISPATCH_N2(g.nx, (assemble_launch<N_>(g, leray, a, nparts, st)));
}

}  // namespace topt
