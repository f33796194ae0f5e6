// rfft.cuh — register-resident line FFT (sm_100a), fp32 (float2) or fp64 (double2).
//
// A line of N = 2^p complex values is held by T = N/E threads, E values each: at entry AND
// at exit thread t holds natural positions t + T*e in a[e] (e < E).  The transform is a
// mixed-radix Stockham FFT (radix E, then the remainder) whose butterflies run in
// registers; only the boundary between two stages goes through shared memory (one write +
// one read of the line), so a 256-point line (16 x 16) costs ONE smem round trip per
// direction instead of one per radix-8 stage plus the staging copies.  Because positions
// coincide at entry and exit, a forward transform, a pointwise spectral multiply and the
// inverse transform chain in registers with no reordering.
//
// Stockham stage (radix R, NS = product of the previous radices, M = N/R): butterfly j takes
// x[j + r M] (r < R), multiplies by W_N^{r k N/(NS R)} with k = j mod NS, runs DFT_R and
// writes x'[(j/NS) NS R + k + q NS] (q < R).  Thread t owns butterflies j = t + b T
// (b < E/R); its inputs are then positions t + T (b + r E/R) — the canonical layout — and
// the outputs of the LAST stage (NS R = N) are positions t + T (b + q E/R), canonical again.
// Twiddles of every stage after the first are loaded once per kernel into registers.
#pragma once
#include "fft.cuh"

namespace topt {

__host__ __device__ constexpr int rf_rad(int N, int E, int ns) { return (N / ns) < E ? N / ns : E; }
// number of register twiddles from stage `ns` on
__host__ __device__ constexpr int rf_ntw(int N, int E, int ns) {
  return ns >= N ? 0 : (ns > 1 ? (E / rf_rad(N, E, ns)) * (rf_rad(N, E, ns) - 1) : 0) + rf_ntw(N, E, ns * rf_rad(N, E, ns));
}
template <int N, int E> struct RfCfg {
  static constexpr int T = N / E;                                   // threads per line
  static constexpr int NTW = rf_ntw(N, E, 1) > 0 ? rf_ntw(N, E, 1) : 1;
  static constexpr int STRIDE = fft_line_stride(N);                 // smem complex per line
};

template <typename C> __device__ __forceinline__ C rf_twid(int N, int m);
template <> __device__ __forceinline__ float2 rf_twid<float2>(int N, int m) { return g_twiddle[N + m]; }
template <> __device__ __forceinline__ double2 rf_twid<double2>(int N, int m) { return g_twiddle_d[N + m]; }

// tw[OFF + b (R-1) + r - 1] = W_N^{r k N/(NS R)}, k = (t + b T) mod NS, for every stage NS > 1
template <int N, int E, int NS, int OFF, typename C>
__device__ __forceinline__ void rf_tw(C* tw, int t) {
  if constexpr (NS < N) {
    constexpr int R = rf_rad(N, E, NS), B = E / R, T = N / E;
    if constexpr (NS > 1) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int k = (t + b * T) & (NS - 1);
#pragma unroll
        for (int r = 1; r < R; ++r) tw[OFF + b * (R - 1) + r - 1] = rf_twid<C>(N, (r * k * (N / (NS * R))) & (N - 1));
      }
      rf_tw<N, E, NS * R, OFF + B * (R - 1), C>(tw, t);
    } else {
      rf_tw<N, E, NS * R, OFF, C>(tw, t);
    }
  }
}

template <bool WARP>
__device__ __forceinline__ void rf_sync() {
  if constexpr (WARP) __syncwarp();
  else __syncthreads();
}

template <int N, int E, int NS, int OFF, bool INV, bool WARP, typename C>
__device__ __forceinline__ void rf_stage(C (&a)[E], C* line, int t, const C* tw) {
  constexpr int R = rf_rad(N, E, NS), B = E / R, T = N / E;
  constexpr bool LAST = NS * R == N;
  C o[E];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    C x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = a[b + r * B];
    if constexpr (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const C w = tw[OFF + b * (R - 1) + r - 1];
        x[r] = INV ? cmulconj(x[r], w) : cmul(x[r], w);
      }
    }
    Dft<R, INV, C>::run(x);
#pragma unroll
    for (int q = 0; q < R; ++q) o[b + q * B] = x[q];
  }
  if constexpr (LAST) {
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = o[e];
  } else {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int j = t + b * T;
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int q = 0; q < R; ++q) line[fft_pad(base + q * NS)] = o[b + q * B];
    }
    rf_sync<WARP>();
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = line[fft_pad(t + T * e)];
    rf_sync<WARP>();
    rf_stage<N, E, NS * R, OFF + (NS > 1 ? B * (R - 1) : 0), INV, WARP, C>(a, line, t, tw);
  }
}

// Unnormalised DFT of the line held in a[] (forward exp(-i k x), inverse exp(+i k x)).
// `line` is this line's smem scratch (RfCfg::STRIDE complex); every thread of the sync
// group (warp if WARP, else block) must call it.
template <int N, int E, bool INV, bool WARP, typename C>
__device__ __forceinline__ void rf_fft(C (&a)[E], C* line, int t, const C* tw) {
  rf_stage<N, E, 1, 0, INV, WARP, C>(a, line, t, tw);
}

}  // namespace topt
