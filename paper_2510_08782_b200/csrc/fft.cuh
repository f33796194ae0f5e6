// fft.cuh — block-cooperative radix-16/8/4/2 Stockham FFT of lines held in shared memory,
// in fp32 (float2) or fp64 (double2) arithmetic.
//
// Used by every spectral kernel of the hot path: the pseudo-spectral derivatives
// (reading R3) and the 3D FFTs of the preconditioner
// (alpha L)^{-1} and of alpha L v.  N = 2^p, 8 <= N <= 1024.
//
// A line of N complex values is transformed in place in shared memory by
// T = max(1, N/16) threads; every stage loads 16 values per thread, applies the
// stage twiddles from a table (host-computed in fp64), runs an in-register DFT of
// radix R = min(16, N/Ns), and writes back in Stockham (auto-sort) order:
//   j in [0, N/R), k = j mod Ns:  a_r = x[j + r N/R] * W^{r k N/(Ns R)},
//   a = DFT_R(a),  x'[(j/Ns) Ns R + k + q Ns] = a_q .
// Shared-memory lines are padded by one element every 16 entries (bank conflicts).
//
// This header DEFINES the device twiddle tables: include it from ONE translation unit.
#pragma once
#include <cuda_runtime.h>

namespace topt {

__host__ __device__ constexpr int fft_threads(int n, int rmax = 16) { return n >= rmax ? n / rmax : 1; }
__host__ __device__ constexpr int fft_pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int fft_line_stride(int n) { return n + n / 16 + 1; }

template <typename C> struct Real;
template <> struct Real<float2> { using T = float; };
template <> struct Real<double2> { using T = double; };

__device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }

template <typename C>
__device__ __forceinline__ C cadd(C a, C b) { return mk(a.x + b.x, a.y + b.y); }
template <typename C>
__device__ __forceinline__ C csub(C a, C b) { return mk(a.x - b.x, a.y - b.y); }
template <typename C>
__device__ __forceinline__ C cmul(C a, C b) { return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }
template <typename C>
__device__ __forceinline__ C cmulconj(C a, C b) { return mk(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)); }
// multiply by -i (forward) or +i (inverse)
template <bool INV, typename C>
__device__ __forceinline__ C mul_mi(C a) { return INV ? mk(-a.y, a.x) : mk(a.y, -a.x); }
// multiply by W = exp(-+ 2 pi i m / R) given cos, sin of 2 pi m / R
template <bool INV, typename C>
__device__ __forceinline__ C mul_w(C a, typename Real<C>::T c, typename Real<C>::T s) {
  return INV ? mk(a.x * c - a.y * s, a.x * s + a.y * c) : mk(a.x * c + a.y * s, a.y * c - a.x * s);
}

template <bool INV, typename C>
__device__ __forceinline__ void dft2(C& a0, C& a1) {
  C t = csub(a0, a1);
  a0 = cadd(a0, a1);
  a1 = t;
}

template <bool INV, typename C>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
  C t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// W_16^m, m = n2*k1 in 0..9 (compile-time after unrolling)
template <bool INV, typename C>
__device__ __forceinline__ C w16(C a, int m) {
  using T = typename Real<C>::T;
  const T c1 = (T)0.92387953251128675613, s1 = (T)0.38268343236508977173, r2 = (T)0.70710678118654752440;
  switch (m & 15) {
    case 0: return a;
    case 1: return mul_w<INV>(a, c1, s1);
    case 2: return mul_w<INV>(a, r2, r2);
    case 3: return mul_w<INV>(a, s1, c1);
    case 4: return mul_mi<INV>(a);
    case 5: return mul_w<INV>(a, -s1, c1);
    case 6: return mul_w<INV>(a, -r2, r2);
    case 7: return mul_w<INV>(a, -c1, s1);
    case 8: return mk(-a.x, -a.y);
    case 9: return mul_w<INV>(a, -c1, -s1);
    default: return a;
  }
}

template <int R, bool INV, typename C>
struct Dft;
template <bool INV, typename C>
struct Dft<1, INV, C> { static __device__ __forceinline__ void run(C*) {} };
template <bool INV, typename C>
struct Dft<2, INV, C> { static __device__ __forceinline__ void run(C* a) { dft2<INV>(a[0], a[1]); } };
template <bool INV, typename C>
struct Dft<4, INV, C> {
  static __device__ __forceinline__ void run(C* a) { dft4<INV>(a[0], a[1], a[2], a[3]); }
};
// 8 = 4 x 2: n = 2 n1 + n2, k = k1 + 4 k2
template <bool INV, typename C>
struct Dft<8, INV, C> {
  static __device__ __forceinline__ void run(C* a) {
    C y0[4] = {a[0], a[2], a[4], a[6]};
    C y1[4] = {a[1], a[3], a[5], a[7]};
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
};
// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
template <bool INV, typename C>
struct Dft<16, INV, C> {
  static __device__ __forceinline__ void run(C* a) {
    C y[4][4];
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
      C b0 = y[0][k1], b1 = y[1][k1], b2 = y[2][k1], b3 = y[3][k1];
      dft4<INV>(b0, b1, b2, b3);
      a[k1] = b0; a[k1 + 4] = b1; a[k1 + 8] = b2; a[k1 + 12] = b3;
    }
  }
};

// One Stockham stage on a padded line `buf`, done by T threads (tid < T).
// tw: table of exp(-2 pi i m / N), m = 0..N-1.
// All threads of the block must call it (it contains __syncthreads); `active` masks work.
template <int N, int R, int NS, bool INV, typename C, int RMAX>
__device__ __forceinline__ void fft_stage(C* buf, const C* tw, int tid, bool active) {
  constexpr int M = N / R;
  constexpr int T = fft_threads(N, RMAX);
  constexpr int NB = M / T;  // butterflies per thread
  C a[NB][R];
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
          const C w = tw[(r * k * (N / (NS * R))) & (N - 1)];
          a[b][r] = INV ? cmulconj(a[b][r], w) : cmul(a[b][r], w);
        }
      }
      Dft<R, INV, C>::run(a[b]);
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

template <int N, int NS, bool INV, typename C, int RMAX>
struct FftStages {
  static __device__ __forceinline__ void run(C* buf, const C* tw, int tid, bool active) {
    constexpr int REM = N / NS;
    constexpr int R = REM >= RMAX ? RMAX : REM;
    fft_stage<N, R, NS, INV, C, RMAX>(buf, tw, tid, active);
    FftStages<N, NS * R, INV, C, RMAX>::run(buf, tw, tid, active);
  }
};
template <int N, bool INV, typename C, int RMAX>
struct FftStages<N, N, INV, C, RMAX> {
  static __device__ __forceinline__ void run(C*, const C*, int, bool) {}
};

// Unnormalised DFT (forward: exp(-i k x), inverse: exp(+i k x)) of a padded smem line by
// fft_threads(N, RMAX) threads (max radix RMAX in {8, 16}).
template <int N, bool INV, int RMAX = 16, typename C>
__device__ __forceinline__ void fft_line(C* buf, const C* tw, int tid, bool active) {
  FftStages<N, 1, INV, C, RMAX>::run(buf, tw, tid, active);
}

// Device twiddle tables: tw[N + m] = exp(-2 pi i m / N), N = 4..1024, computed in fp64
// on the host (upload_twiddles) and rounded once to the table's precision.
__device__ float2 g_twiddle[2048];
__device__ double2 g_twiddle_d[2048];

template <int N>
__device__ __forceinline__ void load_twiddles(float2* s_tw) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_tw[i] = g_twiddle[N + i];
}
template <int N>
__device__ __forceinline__ void load_twiddles(double2* s_tw) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_tw[i] = g_twiddle_d[N + i];
}

}  // namespace topt
