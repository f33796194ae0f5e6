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
  static float2 host[2048];
  for (int N = 4; N <= 1024; N *= 2)
    for (int m = 0; m < N; ++m) {
      const double a = -2.0 * M_PI * (double)m / (double)N;
      host[N + m] = make_float2((float)cos(a), (float)sin(a));
    }
  cudaMemcpyToSymbol(g_twiddle, host, sizeof(host));
}

template <int N>
struct LineCfg {
  static constexpr int T = fft_threads(N);
  static constexpr int LPB = kThreads / T;           // complex lines per 256-thread block
  static constexpr int STRIDE = fft_line_stride(N);  // float2 per smem line
};

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
__global__ void __launch_bounds__(kThreads) k_deriv_x(Geom g, const float* __restrict__ psi,
                                                      size_t psi_stride, const float* __restrict__ lam,
                                                      size_t lam_stride, DerivWeights w, int J,
                                                      float beta, float* __restrict__ out) {
  using C = LineCfg<N>;
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
    fft_line<N, false>(line, tw, tid, active);
    if (active) {
      for (int q = tid; q < N; q += C::T) {
        const float k = kprime(q, N) * invN;
        const float2 z = line[fft_pad(q)];
        line[fft_pad(q)] = make_float2(-k * z.y, k * z.x);  // i k' z / N
      }
    }
    __syncthreads();
    fft_line<N, true>(line, tw, tid, active);
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
__global__ void __launch_bounds__(kThreads) k_deriv_strided(Geom g, int axis, int TX,
                                                            const float* __restrict__ psi,
                                                            size_t psi_stride,
                                                            const float* __restrict__ lam,
                                                            size_t lam_stride, DerivWeights w, int J,
                                                            float beta, float* __restrict__ out) {
  using C = LineCfg<N>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  const int nlines = TX / 2;
  const int tilesx = g.nx / TX;
  const int x0 = (blockIdx.x % tilesx) * TX;
  const int outer = blockIdx.x / tilesx;
  size_t base, S;
  if (axis == 1) { base = ((size_t)outer << (g.lx + g.ly)) + x0; S = g.nx; }
  else { base = ((size_t)outer << g.lx) + x0; S = (size_t)g.nx * g.ny; }
  const int TX4 = TX / 4;
  const int n4 = N * TX4;  // float4 in the tile
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  const bool active = myline < nlines;
  constexpr int MAXE = 8;  // N*TX/4 / (TX/2 * T) = N/(2T) <= 8
  float4 acc[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float invN = 1.0f / (float)N;
  const int nthreads = blockDim.x;
  for (int j = 0; j < J; ++j) {
    const float* src = psi + j * psi_stride;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int f4 = threadIdx.x + e * nthreads;
      if (f4 >= n4) break;
      const int row = f4 / TX4, c4 = f4 % TX4;
      const float4 val = *reinterpret_cast<const float4*>(src + base + row * S + c4 * 4);
      float* l0 = reinterpret_cast<float*>(buf + (2 * c4) * C::STRIDE + fft_pad(row));
      float* l1 = reinterpret_cast<float*>(buf + (2 * c4 + 1) * C::STRIDE + fft_pad(row));
      l0[0] = val.x; l0[1] = val.y; l1[0] = val.z; l1[1] = val.w;
    }
    __syncthreads();
    float2* line = buf + myline * C::STRIDE;
    fft_line<N, false>(line, tw, tid, active);
    if (active) {
      for (int q = tid; q < N; q += C::T) {
        const float k = kprime(q, N) * invN;
        const float2 z = line[fft_pad(q)];
        line[fft_pad(q)] = make_float2(-k * z.y, k * z.x);
      }
    }
    __syncthreads();
    fft_line<N, true>(line, tw, tid, active);
    const float wj = w.w[j];
    const float* lj = lam ? lam + j * lam_stride : nullptr;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int f4 = threadIdx.x + e * nthreads;
      if (f4 >= n4) break;
      const int row = f4 / TX4, c4 = f4 % TX4;
      const float2 d0 = buf[(2 * c4) * C::STRIDE + fft_pad(row)];
      const float2 d1 = buf[(2 * c4 + 1) * C::STRIDE + fft_pad(row)];
      float4 l4 = make_float4(1.f, 1.f, 1.f, 1.f);
      if (lj) l4 = *reinterpret_cast<const float4*>(lj + base + row * S + c4 * 4);
      acc[e].x = fmaf(wj * l4.x, d0.x, acc[e].x);
      acc[e].y = fmaf(wj * l4.y, d0.y, acc[e].y);
      acc[e].z = fmaf(wj * l4.z, d1.x, acc[e].z);
      acc[e].w = fmaf(wj * l4.w, d1.y, acc[e].w);
    }
  }
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int f4 = threadIdx.x + e * nthreads;
    if (f4 >= n4) break;
    const int row = f4 / TX4, c4 = f4 % TX4;
    float4* o = reinterpret_cast<float4*>(out + base + row * S + c4 * 4);
    float4 r = acc[e];
    if (beta != 0.0f) {
      const float4 p = *o;
      r.x += beta * p.x; r.y += beta * p.y; r.z += beta * p.z; r.w += beta * p.w;
    }
    *o = r;
  }
}

template <int N>
static size_t line_smem() {
  using C = LineCfg<N>;
  return (size_t)(C::LPB * C::STRIDE + N) * sizeof(float2);
}

template <int N>
static void deriv_dispatch(const Geom& g, int axis, const DerivArgs& a, const DerivWeights& w,
                           cudaStream_t st) {
  using C = LineCfg<N>;
  const size_t sm = line_smem<N>();
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
// Preconditioner passes.
// =====================================================================================

// Forward x pass: Z[row][pos(q)] = FFT_x(v + i b)[q]   (rows = ny*nz, one complex line per row)
template <int N>
__global__ void __launch_bounds__(kThreads) k_px_fwd(Geom g, const float* __restrict__ v,
                                                     const float* __restrict__ b,
                                                     float2* __restrict__ Z) {
  using C = LineCfg<N>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  const size_t nrows = (size_t)g.ny * g.nz;
  const size_t row0 = (size_t)blockIdx.x * C::LPB;
  const int comp = blockIdx.y;
  const float* vc = v ? v + comp * g.F : nullptr;
  const float* bc = b ? b + comp * g.F : nullptr;
  float2* Zc = Z + comp * g.F;
  const int n4 = C::LPB * N / 4;
  for (int f4 = threadIdx.x; f4 < n4; f4 += kThreads) {
    const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
    const size_t gi = (row0 + rl) * N + pos;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
    if (row0 + rl < nrows) {
      if (vc) a = *reinterpret_cast<const float4*>(vc + gi);
      if (bc) c = *reinterpret_cast<const float4*>(bc + gi);
    }
    float2* L = buf + rl * C::STRIDE;
    L[fft_pad(pos + 0)] = make_float2(a.x, c.x);
    L[fft_pad(pos + 1)] = make_float2(a.y, c.y);
    L[fft_pad(pos + 2)] = make_float2(a.z, c.z);
    L[fft_pad(pos + 3)] = make_float2(a.w, c.w);
  }
  __syncthreads();
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  fft_line<N, false>(buf + myline * C::STRIDE, tw, tid, myline < C::LPB);
  for (int i = threadIdx.x; i < C::LPB * N; i += kThreads) {
    const int rl = i / N, p = i % N;
    if (row0 + rl < nrows) Zc[(row0 + rl) * N + p] = buf[rl * C::STRIDE + fft_pad(paired_q(p, N))];
  }
}

// Inverse x pass: g + i s = IFFT_x(Z) (paired order in), reductions max|g|, sum g*s.
template <int N>
__global__ void __launch_bounds__(kThreads) k_px_inv(Geom g, const float2* __restrict__ Z,
                                                     float* __restrict__ gout, float* __restrict__ sout,
                                                     double* __restrict__ partials, int pstride) {
  using C = LineCfg<N>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  const size_t nrows = (size_t)g.ny * g.nz;
  const size_t row0 = (size_t)blockIdx.x * C::LPB;
  const int comp = blockIdx.y;
  const float2* Zc = Z + comp * g.F;
  for (int i = threadIdx.x; i < C::LPB * N; i += kThreads) {
    const int rl = i / N, p = i % N;
    float2 z = make_float2(0.f, 0.f);
    if (row0 + rl < nrows) z = Zc[(row0 + rl) * N + p];
    buf[rl * C::STRIDE + fft_pad(paired_q(p, N))] = z;
  }
  __syncthreads();
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  fft_line<N, true>(buf + myline * C::STRIDE, tw, tid, myline < C::LPB);
  double gmax = 0.0, gs = 0.0;
  const int n4 = C::LPB * N / 4;
  for (int f4 = threadIdx.x; f4 < n4; f4 += kThreads) {
    const int rl = (f4 * 4) / N, pos = (f4 * 4) % N;
    if (row0 + rl >= nrows) continue;
    const size_t gi = comp * g.F + (row0 + rl) * N + pos;
    const float2* L = buf + rl * C::STRIDE;
    const float2 a0 = L[fft_pad(pos)], a1 = L[fft_pad(pos + 1)], a2 = L[fft_pad(pos + 2)],
                 a3 = L[fft_pad(pos + 3)];
    if (gout) *reinterpret_cast<float4*>(gout + gi) = make_float4(a0.x, a1.x, a2.x, a3.x);
    if (sout) *reinterpret_cast<float4*>(sout + gi) = make_float4(a0.y, a1.y, a2.y, a3.y);
    gmax = fmax(gmax, (double)fmaxf(fmaxf(fabsf(a0.x), fabsf(a1.x)), fmaxf(fabsf(a2.x), fabsf(a3.x))));
    gs += (double)(a0.x * a0.y) + (double)(a1.x * a1.y) + (double)(a2.x * a2.y) + (double)(a3.x * a3.y);
  }
  // block reductions (max, sum) in fixed order
  __shared__ double shm[32], shs[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gmax = fmax(gmax, __shfl_down_sync(0xffffffffu, gmax, o));
    gs += __shfl_down_sync(0xffffffffu, gs, o);
  }
  if ((threadIdx.x & 31) == 0) { shm[threadIdx.x >> 5] = gmax; shs[threadIdx.x >> 5] = gs; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0, s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) { m = fmax(m, shm[w]); s += shs[w]; }
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    partials[bid] = m;
    partials[pstride + bid] = s;
  }
}

// Middle (y) pass of the 3D FFT, in place.  INV = false: natural in, paired out.
// INV = true: paired in, natural out.  Tile: TXC complex columns x N rows at fixed z.
template <int N, bool INV>
__global__ void __launch_bounds__(kThreads) k_py(Geom g, int TXC, float2* __restrict__ Z) {
  using C = LineCfg<N>;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* tw = smem + C::LPB * C::STRIDE;
  load_twiddles<N>(tw);
  const int tilesx = g.nx / TXC;
  const int x0 = (blockIdx.x % tilesx) * TXC;
  const int z = blockIdx.x / tilesx;
  float2* Zc = Z + blockIdx.y * g.F + ((size_t)z << (g.lx + g.ly)) + x0;
  const int n = N * TXC;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = i / TXC, c = i % TXC;
    const int q = INV ? paired_q(row, N) : row;
    buf[c * C::STRIDE + fft_pad(q)] = Zc[(size_t)row * g.nx + c];
  }
  __syncthreads();
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  fft_line<N, INV>(buf + myline * C::STRIDE, tw, tid, myline < TXC);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = i / TXC, c = i % TXC;
    const int q = INV ? row : paired_q(row, N);
    Zc[(size_t)row * g.nx + c] = buf[c * C::STRIDE + fft_pad(q)];
  }
}

struct SpecParams {
  float alpha;
  int p;
  int leray;
  int ncomp;      // components processed per block (d if leray, else 1)
  float invn;     // 1 / (nx ny nz)
};

__device__ __forceinline__ float regL(float kk, int p) {
  return p == 1 ? kk : (p == 2 ? kk * kk : kk * kk * kk);
}

// Fused last-axis pass: forward FFT along the last axis, spectral operator, inverse FFT.
// 3D: tile = TXC x-positions (even) x 2 y-positions {2m, 2m+1} x N_z, for `ncomp` comps.
// 2D: tile = TXC x-positions x N_y.
// Spectral operator on each pair (k, -k):  v^ = (Z(k) + conj Z(-k))/2,
// b^ = (Z(k) - conj Z(-k))/(2i), g^ = alpha L v^ + b^ (P_L g^ if leray),
// s^ = -g^/(alpha L~), Z(k) <- (g^ + i s^)/n.  Partials: L|v^|^2, Re(s^ conj(L v^)), L|s^|^2.
template <int N, int D>
__global__ void __launch_bounds__(768) k_plast(Geom g, int TXC, SpecParams sp, float2* __restrict__ Z,
                                               double* __restrict__ partials, int pstride) {
  using C = LineCfg<N>;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* buf = smem + N;
  load_twiddles<N>(tw);
  const int ny2 = D == 3 ? 2 : 1;                 // y-positions per tile
  const int lines_per_comp = TXC * ny2;
  const int nlines = lines_per_comp * sp.ncomp;
  const int tilesx = g.nx / TXC;
  const int x0 = (blockIdx.x % tilesx) * TXC;
  const int y0 = D == 3 ? (blockIdx.x / tilesx) * 2 : 0;
  const int comp0 = sp.ncomp == 1 ? blockIdx.y : 0;
  const size_t S = D == 3 ? (size_t)g.nx * g.ny : (size_t)g.nx;  // stride along the last axis
  // line l: comp = l / lines_per_comp, r = l % lines_per_comp, yy = r / TXC, c = r % TXC
  auto gptr = [&](int l) -> float2* {
    const int comp = comp0 + l / lines_per_comp, r = l % lines_per_comp;
    const int yy = r / TXC, c = r % TXC;
    return Z + comp * g.F + (size_t)(y0 + yy) * g.nx + x0 + c;
  };
  const int n = N * nlines;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = i / nlines, l = i % nlines;
    buf[l * C::STRIDE + fft_pad(row)] = gptr(l)[row * S];
  }
  __syncthreads();
  const int myline = threadIdx.x / C::T, tid = threadIdx.x % C::T;
  const bool active = myline < nlines;
  fft_line<N, false>(buf + myline * C::STRIDE, tw, tid, active);

  // spectral operator over points of one component-set: pt = (r, qz), r in [0, lines_per_comp)
  double s_reg = 0.0, s_slv = 0.0, s_sls = 0.0;
  const int npts = lines_per_comp * N;
  const float al = sp.alpha;
  for (int pt = threadIdx.x; pt < npts; pt += blockDim.x) {
    const int r = pt / N, qz = pt % N;
    const int yy = r / TXC, c = r % TXC;
    const int xp = x0 + c, yp = y0 + yy;
    // partner position
    const int xpp = xp < 2 ? xp : (xp ^ 1);
    const int ypp = D == 3 ? (yp < 2 ? yp : (yp ^ 1)) : 0;
    const int qzp = (N - qz) & (N - 1);
    const int rp = (ypp - y0) * TXC + (xpp - x0);
    const int pt2 = rp * N + qzp;
    if (pt2 < pt) continue;  // the partner's thread handles the pair
    const bool self = pt2 == pt;
    // wavenumbers (R2, R3)
    const int qx = paired_q(xp, g.nx);
    const float kx = kfreq(qx, g.nx), kpx = kprime(qx, g.nx);
    float ky, kpy, kz, kpz;
    if (D == 3) {
      const int qy = paired_q(yp, g.ny);
      ky = kfreq(qy, g.ny); kpy = kprime(qy, g.ny);
      kz = kfreq(qz, N); kpz = kprime(qz, N);
    } else {
      ky = kfreq(qz, N); kpy = kprime(qz, N);
      kz = 0.f; kpz = 0.f;
    }
    const float kk = kx * kx + ky * ky + kz * kz;
    const float L = regL(kk, sp.p);
    const float Lt = L == 0.f ? 1.f : L;  // kernel fix
    float2 gh[3], vh[3];
    for (int cc = 0; cc < sp.ncomp; ++cc) {
      const float2 z1 = buf[(cc * lines_per_comp + r) * C::STRIDE + fft_pad(qz)];
      const float2 z2 = buf[(cc * lines_per_comp + rp) * C::STRIDE + fft_pad(qzp)];
      const float2 v1 = make_float2(0.5f * (z1.x + z2.x), 0.5f * (z1.y - z2.y));
      // b^ = (z1 - conj z2) / (2i) = -i/2 (z1 - conj z2)
      const float2 dd = make_float2(z1.x - z2.x, z1.y + z2.y);
      const float2 b1 = make_float2(0.5f * dd.y, -0.5f * dd.x);
      vh[cc] = v1;
      gh[cc] = make_float2(fmaf(al * L, v1.x, b1.x), fmaf(al * L, v1.y, b1.y));
    }
    if (sp.leray) {
      const float kp2 = kpx * kpx + kpy * kpy + kpz * kpz;
      if (kp2 > 0.f) {
        const float kp[3] = {kpx, kpy, kpz};
        float2 dot = make_float2(0.f, 0.f);
        for (int cc = 0; cc < sp.ncomp; ++cc) { dot.x += kp[cc] * gh[cc].x; dot.y += kp[cc] * gh[cc].y; }
        const float inv = 1.0f / kp2;
        for (int cc = 0; cc < sp.ncomp; ++cc) {
          gh[cc].x -= kp[cc] * dot.x * inv;
          gh[cc].y -= kp[cc] * dot.y * inv;
        }
      }
    }
    const float invaL = 1.0f / (al * Lt);
    const double mult = self ? 1.0 : 2.0;
    for (int cc = 0; cc < sp.ncomp; ++cc) {
      const float2 gg = gh[cc];
      const float2 ss = make_float2(-gg.x * invaL, -gg.y * invaL);
      const float2 vv = vh[cc];
      s_reg += mult * (double)L * ((double)vv.x * vv.x + (double)vv.y * vv.y);
      s_slv += mult * (double)L * ((double)ss.x * vv.x + (double)ss.y * vv.y);
      s_sls += mult * (double)L * ((double)ss.x * ss.x + (double)ss.y * ss.y);
      // W(k) = (g^ + i s^)/n ; W(-k) = (conj g^ + i conj s^)/n
      const float in = sp.invn;
      buf[(cc * lines_per_comp + r) * C::STRIDE + fft_pad(qz)] =
          make_float2((gg.x - ss.y) * in, (gg.y + ss.x) * in);
      if (!self)
        buf[(cc * lines_per_comp + rp) * C::STRIDE + fft_pad(qzp)] =
            make_float2((gg.x + ss.y) * in, (-gg.y + ss.x) * in);
    }
  }
  __syncthreads();
  fft_line<N, true>(buf + myline * C::STRIDE, tw, tid, active);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = i / nlines, l = i % nlines;
    gptr(l)[row * S] = buf[l * C::STRIDE + fft_pad(row)];
  }
  // partial sums
  __shared__ double sh[3][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s_reg += __shfl_down_sync(0xffffffffu, s_reg, o);
    s_slv += __shfl_down_sync(0xffffffffu, s_slv, o);
    s_sls += __shfl_down_sync(0xffffffffu, s_sls, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = s_reg; sh[1][threadIdx.x >> 5] = s_slv; sh[2][threadIdx.x >> 5] = s_sls;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) { a += sh[0][w]; b += sh[1][w]; c += sh[2][w]; }
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    partials[bid] = a;
    partials[pstride + bid] = b;
    partials[2 * pstride + bid] = c;
  }
}

template <int N>
static void px_fwd_dispatch(const Geom& g, const PrecondArgs& a, cudaStream_t st) {
  using C = LineCfg<N>;
  const size_t sm = line_smem<N>();
  const size_t nrows = (size_t)g.ny * g.nz;
  dim3 grid((unsigned)((nrows + C::LPB - 1) / C::LPB), g.d);
  cudaFuncSetAttribute(k_px_fwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_px_fwd<N><<<grid, kThreads, sm, st>>>(g, a.v, a.b, a.Z);
}

template <int N>
static void px_inv_dispatch(const Geom& g, const PrecondArgs& a, int* nparts, cudaStream_t st) {
  using C = LineCfg<N>;
  const size_t sm = line_smem<N>();
  const size_t nrows = (size_t)g.ny * g.nz;
  dim3 grid((unsigned)((nrows + C::LPB - 1) / C::LPB), g.d);
  *nparts = grid.x * grid.y;
  cudaFuncSetAttribute(k_px_inv<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_px_inv<N><<<grid, kThreads, sm, st>>>(g, a.Z, a.g, a.s, a.partials + 3 * kMaxPartials,
                                          kMaxPartials);
}

template <int N>
static void py_dispatch(const Geom& g, bool inv, const PrecondArgs& a, cudaStream_t st) {
  using C = LineCfg<N>;
  const size_t sm = line_smem<N>();
  int TXC = C::LPB < g.nx ? C::LPB : g.nx;
  dim3 grid((g.nx / TXC) * g.nz, g.d);
  const int threads = TXC * C::T;
  if (inv) {
    cudaFuncSetAttribute(k_py<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_py<N, true><<<grid, threads, sm, st>>>(g, TXC, a.Z);
  } else {
    cudaFuncSetAttribute(k_py<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_py<N, false><<<grid, threads, sm, st>>>(g, TXC, a.Z);
  }
}

template <int N>
static void plast_dispatch(const Geom& g, const PrecondArgs& a, int* nparts, cudaStream_t st) {
  using C = LineCfg<N>;
  SpecParams sp;
  sp.alpha = (float)a.alpha;
  sp.p = a.p;
  sp.leray = a.leray ? 1 : 0;
  sp.ncomp = a.leray ? g.d : 1;
  sp.invn = (float)(1.0 / ((double)g.nx * g.ny * g.nz));
  const int ny2 = g.d == 3 ? 2 : 1;
  // lines per block target ~ LPB (256 threads); at least 2 x-positions per tile
  int TXC = C::LPB / (ny2 * sp.ncomp);
  int t = 2;
  while (t * 2 <= TXC) t *= 2;
  TXC = t < 2 ? 2 : t;
  if (TXC > g.nx) TXC = g.nx;
  const int nlines = TXC * ny2 * sp.ncomp;
  const int threads = nlines * C::T;
  const size_t sm = (size_t)(N + nlines * C::STRIDE) * sizeof(float2);
  const int tiles = (g.nx / TXC) * (g.d == 3 ? g.ny / 2 : 1);
  dim3 grid(tiles, sp.ncomp == 1 ? g.d : 1);
  *nparts = grid.x * grid.y;
  double* part = a.partials;
  if (g.d == 3) {
    cudaFuncSetAttribute(k_plast<N, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_plast<N, 3><<<grid, threads, sm, st>>>(g, TXC, sp, a.Z, part, kMaxPartials);
  } else {
    cudaFuncSetAttribute(k_plast<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_plast<N, 2><<<grid, threads, sm, st>>>(g, TXC, sp, a.Z, part, kMaxPartials);
  }
}

// Full preconditioner: 3D: x, y, [z fused], y^-1, x^-1;  2D: x, [y fused], x^-1.
// Scalars written: REG, SLV, SLS (spectral, h^d/n weighted), GRAD_INF, GS (real space).
void launch_precond(const Geom& g, const PrecondArgs& a, cudaStream_t st) {
  TOPT_DISPATCH_N(g.nx, px_fwd_dispatch, g, a, st);
  if (g.d == 3) TOPT_DISPATCH_N(g.ny, py_dispatch, g, false, a, st);
  int np_last = 0, np_inv = 0;
  const int Nl = g.d == 3 ? g.nz : g.ny;
  TOPT_DISPATCH_N(Nl, plast_dispatch, g, a, &np_last, st);
  if (g.d == 3) TOPT_DISPATCH_N(g.ny, py_dispatch, g, true, a, st);
  TOPT_DISPATCH_N(g.nx, px_inv_dispatch, g, a, &np_inv, st);
  if (a.scalars) {
    const double n = (double)g.F;
    const double sc = a.cellvol / n;  // Parseval: <a,b>_h = h^d/n sum_k a^ conj b^
    launch_finalize(a.partials, 0, np_last, 0.5 * a.alpha * sc, false, a.scalars + TOPT_S_REG, st);
    launch_finalize(a.partials, 1, np_last, a.alpha * sc, false, a.scalars + TOPT_S_SLV, st);
    launch_finalize(a.partials, 2, np_last, a.alpha * sc, false, a.scalars + TOPT_S_SLS, st);
    launch_finalize(a.partials, 3, np_inv, 1.0, true, a.scalars + TOPT_S_GRAD_INF, st);
    launch_finalize(a.partials, 4, np_inv, a.cellvol, false, a.scalars + TOPT_S_GS, st);
  }
}

}  // namespace topt
