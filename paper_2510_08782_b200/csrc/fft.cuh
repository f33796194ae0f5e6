// fft.cuh — block-cooperative radix-16/8/4/2 Stockham FFT of lines held in shared memory.
//
// Used by every spectral kernel of the hot path: the pseudo-spectral derivatives
// (reading R3) and the 3D FFT of the preconditioner
// (alpha L)^{-1}.  N = 2^p, 4 <= N <= 1024.
//
// A line of N complex values is transformed in place in shared memory by
// T = max(1, N/16) threads; every stage loads 16 values per thread, applies the
// stage twiddles from a table (host-computed in fp64), runs an in-register DFT of
// radix R = min(16, N/Ns), and writes back in Stockham (auto-sort) order:
//   j in [0, N/R), k = j mod Ns:  a_r = x[j + r N/R] * W^{r k N/(Ns R)},
//   a = DFT_R(a),  x'[(j/Ns) Ns R + k + q Ns] = a_q .
// Shared memory lines are padded by one float2 every 16 entries (bank conflicts).
#pragma once
#include <cuda_runtime.h>

namespace topt {

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int fft_threads(int n) { return n >= 16 ? n / 16 : 1; }
__host__ __device__ constexpr int fft_pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int fft_line_stride(int n) { return n + n / 16 + 1; }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulconj(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
// multiply by W_R^m = exp(-+ 2 pi i m / R) given cos/sin of 2 pi m / R
template <bool INV>
__device__ __forceinline__ float2 mul_w(float2 a, float c, float s) {
  return INV ? make_float2(a.x * c - a.y * s, a.x * s + a.y * c)
             : make_float2(a.x * c + a.y * s, a.y * c - a.x * s);
}

template <bool INV>
__device__ __forceinline__ void dft2(float2& a0, float2& a1) {
  float2 t = csub(a0, a1);
  a0 = cadd(a0, a1);
  a1 = t;
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  float2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// cos / sin (2 pi m / 16), m = 0..15
#define TOPT_C16_1 0.92387953251128674f
#define TOPT_S16_1 0.38268343236508978f
#define TOPT_R2 0.70710678118654752f

template <bool INV>
__device__ __forceinline__ float2 w16(float2 a, int m) {  // m compile-time after unrolling
  switch (m & 15) {
    case 0: return a;
    case 1: return mul_w<INV>(a, TOPT_C16_1, TOPT_S16_1);
    case 2: return mul_w<INV>(a, TOPT_R2, TOPT_R2);
    case 3: return mul_w<INV>(a, TOPT_S16_1, TOPT_C16_1);
    case 4: return mul_mi<INV>(a);
    case 5: return mul_w<INV>(a, -TOPT_S16_1, TOPT_C16_1);
    case 6: return mul_w<INV>(a, -TOPT_R2, TOPT_R2);
    case 7: return mul_w<INV>(a, -TOPT_C16_1, TOPT_S16_1);
    case 8: return make_float2(-a.x, -a.y);
    case 9: return mul_w<INV>(a, -TOPT_C16_1, -TOPT_S16_1);
    default: return a;  // not reached for radix 16 (n2*k1 <= 9)
  }
}

// In-register DFT of size R on a[0..R-1], natural order in and out.
template <int R, bool INV>
__device__ __forceinline__ void dft(float2* a);

template <>
__device__ __forceinline__ void dft<1, false>(float2*) {}
template <>
__device__ __forceinline__ void dft<1, true>(float2*) {}
template <>
__device__ __forceinline__ void dft<2, false>(float2* a) { dft2<false>(a[0], a[1]); }
template <>
__device__ __forceinline__ void dft<2, true>(float2* a) { dft2<true>(a[0], a[1]); }
template <>
__device__ __forceinline__ void dft<4, false>(float2* a) { dft4<false>(a[0], a[1], a[2], a[3]); }
template <>
__device__ __forceinline__ void dft<4, true>(float2* a) { dft4<true>(a[0], a[1], a[2], a[3]); }

// 8 = 4 x 2: n = 2 n1 + n2, k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft8_impl(float2* a) {
  float2 y0[4] = {a[0], a[2], a[4], a[6]};
  float2 y1[4] = {a[1], a[3], a[5], a[7]};
  dft4<INV>(y0[0], y0[1], y0[2], y0[3]);
  dft4<INV>(y1[0], y1[1], y1[2], y1[3]);
  y1[1] = w16<INV>(y1[1], 2);
  y1[2] = w16<INV>(y1[2], 4);
  y1[3] = w16<INV>(y1[3], 6);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    a[k1] = cadd(y0[k1], y1[k1]);
    a[k1 + 4] = csub(y0[k1], y1[k1]);
  }
}
template <>
__device__ __forceinline__ void dft<8, false>(float2* a) { dft8_impl<false>(a); }
template <>
__device__ __forceinline__ void dft<8, true>(float2* a) { dft8_impl<true>(a); }

// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft16_impl(float2* a) {
  float2 y[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    y[n2][0] = a[n2]; y[n2][1] = a[4 + n2]; y[n2][2] = a[8 + n2]; y[n2][3] = a[12 + n2];
    dft4<INV>(y[n2][0], y[n2][1], y[n2][2], y[n2][3]);
  }
#pragma unroll
  for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) y[n2][k1] = w16<INV>(y[n2][k1], n2 * k1);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 b0 = y[0][k1], b1 = y[1][k1], b2 = y[2][k1], b3 = y[3][k1];
    dft4<INV>(b0, b1, b2, b3);
    a[k1] = b0; a[k1 + 4] = b1; a[k1 + 8] = b2; a[k1 + 12] = b3;
  }
}
template <>
__device__ __forceinline__ void dft<16, false>(float2* a) { dft16_impl<false>(a); }
template <>
__device__ __forceinline__ void dft<16, true>(float2* a) { dft16_impl<true>(a); }

// One Stockham stage on a padded line `buf` (stride fft_pad), done by T threads (tid < T).
// tw: table of exp(-2 pi i m / N), m = 0..N-1 (padded indexing not used for the table).
// All threads of the block must call it (it contains __syncthreads) — `active` masks work.
template <int N, int R, int NS, bool INV>
__device__ __forceinline__ void fft_stage(float2* buf, const float2* tw, int tid, bool active) {
  constexpr int M = N / R;
  constexpr int T = fft_threads(N);
  constexpr int NB = M / T;  // butterflies per thread
  float2 a[NB][R];
  if (active) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = tid + b * T;
      const int k = j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) a[b][r] = buf[fft_pad(j + r * M)];
      if (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const float2 w = tw[(r * k * (N / (NS * R))) & (N - 1)];
          a[b][r] = INV ? cmulconj(a[b][r], w) : cmul(a[b][r], w);
        }
      }
      dft<R, INV>(a[b]);
    }
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = tid + b * T;
      const int k = j % NS;
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[fft_pad(base + r * NS)] = a[b][r];
    }
  }
  __syncthreads();
}

template <int N, int NS, bool INV>
struct FftStages {
  static __device__ __forceinline__ void run(float2* buf, const float2* tw, int tid, bool active) {
    constexpr int REM = N / NS;
    constexpr int R = REM >= 16 ? 16 : REM;
    fft_stage<N, R, NS, INV>(buf, tw, tid, active);
    FftStages<N, NS * R, INV>::run(buf, tw, tid, active);
  }
};
template <int N, bool INV>
struct FftStages<N, N, INV> {
  static __device__ __forceinline__ void run(float2*, const float2*, int, bool) {}
};

// Unnormalised DFT (forward: exp(-i k x), inverse: exp(+i k x)) of a padded smem line.
template <int N, bool INV>
__device__ __forceinline__ void fft_line(float2* buf, const float2* tw, int tid, bool active) {
  FftStages<N, 1, INV>::run(buf, tw, tid, active);
}

// Device twiddle tables: g_twiddle[N + m] = exp(-2 pi i m / N) for N = 4..1024 (fp64-rounded),
// filled by upload_twiddles(). Defined here: include this header from ONE translation unit.
__device__ float2 g_twiddle[2048];

// Copy the twiddle table of size N into shared memory (all threads).
template <int N>
__device__ __forceinline__ void load_twiddles(float2* s_tw) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_tw[i] = g_twiddle[N + i];
}

}  // namespace topt
