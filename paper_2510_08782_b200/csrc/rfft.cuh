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
// Twiddles: per stage after the first and per butterfly, only the base powers W^m, W^2m,
// W^4m, W^8m (m = k N/(NS R), the ones below R) are loaded once per kernel into registers
// (from the fp64-computed table); the other powers are composed on the fly, each a product
// of at most three bases, so an fp32 twiddle carries at most a few ulps.
#pragma once
#include "fft.cuh"

namespace topt {

__host__ __device__ constexpr int rf_rad(int N, int E, int ns) { return (N / ns) < E ? N / ns : E; }
// twiddles kept per butterfly for radix R: all R-1 powers (FULL), or the base powers W^m
// (R >= 2), W^2m (R >= 4), W^4m (R >= 8), W^8m (R >= 16)
__host__ __device__ constexpr int rf_nb(int R, bool full) {
  return full ? R - 1 : (R >= 16 ? 4 : (R >= 8 ? 3 : (R >= 4 ? 2 : 1)));
}
// number of register twiddles from stage `ns` on
__host__ __device__ constexpr int rf_ntw(int N, int E, int ns, bool full) {
  return ns >= N ? 0
                 : (ns > 1 ? (E / rf_rad(N, E, ns)) * rf_nb(rf_rad(N, E, ns), full) : 0) +
                       rf_ntw(N, E, ns * rf_rad(N, E, ns), full);
}
template <int N, int E, bool FULL = false> struct RfCfg {
  static constexpr int T = N / E;                                   // threads per line
  static constexpr int NTW = rf_ntw(N, E, 1, FULL) > 0 ? rf_ntw(N, E, 1, FULL) : 1;
  static constexpr int STRIDE = fft_line_stride(N);                 // smem complex per line
};

template <typename C> __device__ __forceinline__ C rf_twid(int N, int m);
template <> __device__ __forceinline__ float2 rf_twid<float2>(int N, int m) { return g_twiddle[N + m]; }
template <> __device__ __forceinline__ double2 rf_twid<double2>(int N, int m) { return g_twiddle_d[N + m]; }

// For every stage NS > 1 and butterfly b (m = k N/(NS R), k = (t + b T) mod NS):
// FULL: tw[OFF + b (R-1) + r - 1] = W_N^{r m}; else tw[OFF + b nb + i] = W_N^{2^i m}.
template <int N, int E, int NS, int OFF, bool FULL, typename C>
__device__ __forceinline__ void rf_tw(C* tw, int t) {
  if constexpr (NS < N) {
    constexpr int R = rf_rad(N, E, NS), B = E / R, T = N / E, NB = rf_nb(R, FULL);
    if constexpr (NS > 1) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int m = ((t + b * T) & (NS - 1)) * (N / (NS * R));
#pragma unroll
        for (int i = 0; i < NB; ++i)
          tw[OFF + b * NB + i] = rf_twid<C>(N, (FULL ? (i + 1) * m : (m << i)) & (N - 1));
      }
      rf_tw<N, E, NS * R, OFF + B * NB, FULL, C>(tw, t);
    } else {
      rf_tw<N, E, NS * R, OFF, FULL, C>(tw, t);
    }
  }
}
template <int N, int E, bool FULL = false, typename C>
__device__ __forceinline__ void rf_twiddles(C* tw, int t) {
  rf_tw<N, E, 1, 0, FULL, C>(tw, t);
}

// w[r] = W^{r m} for r = 1 .. R-1 from the bases w1 = W^m, w2, w4, w8 (at most 3 products deep)
template <int R, typename C>
__device__ __forceinline__ void rf_powers(const C* base, C* w) {
  w[1] = base[0];
  if constexpr (R > 2) {
    w[2] = base[1];
    w[3] = cmul(w[2], w[1]);
  }
  if constexpr (R > 4) {
    w[4] = base[2];
    w[5] = cmul(w[4], w[1]);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
  }
  if constexpr (R > 8) {
    w[8] = base[3];
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[8], w[r - 8]);
  }
}

template <bool WARP>
__device__ __forceinline__ void rf_sync() {
  if constexpr (WARP) __syncwarp();
  else __syncthreads();
}

// scratch addressing of the stage-boundary exchange: LS == 0 -> line[fft_pad(i)] (a padded line of
// its own); LS > 0 -> line[i * LS] (lines interleaved with stride LS: a [position][line] tile, e.g. a
// TMA-staged input tile reused as scratch once its values are in registers)
// In the interleaved form a phase of a warp's accesses holds several positions of each column; the
// first stage's writes put neighbouring threads' positions E apart (radix E: same parity, same
// banks), so position i is stored at i ^ bit_log2(E)(i) — a bijection that gives them different
// parities.  SH = log2(E).
#ifndef TOPT_RF_SWZ
#define TOPT_RF_SWZ 1
#endif
template <int LS, int SH>
__device__ __forceinline__ int rf_idx(int i) {
  return LS == 0 ? fft_pad(i) : (TOPT_RF_SWZ ? (i ^ ((i >> SH) & 1)) : i) * LS;
}
__host__ __device__ constexpr int rf_log2(int e) { return e <= 1 ? 0 : 1 + rf_log2(e / 2); }

template <int N, int E, int NS, int OFF, bool INV, bool WARP, bool FULL, int LS, typename C>
__device__ __forceinline__ void rf_stage(C (&a)[E], C* line, int t, const C* tw) {
  constexpr int R = rf_rad(N, E, NS), B = E / R, T = N / E, NB = rf_nb(R, FULL);
  constexpr bool LAST = NS * R == N;
  C o[E];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    C x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = a[b + r * B];
    if constexpr (NS > 1) {
      C w[R];
      if constexpr (FULL) {
#pragma unroll
        for (int r = 1; r < R; ++r) w[r] = tw[OFF + b * NB + r - 1];
      } else {
        rf_powers<R>(tw + OFF + b * NB, w);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) x[r] = INV ? cmulconj(x[r], w[r]) : cmul(x[r], w[r]);
    }
    Dft<R, INV, C>::run(x);
#pragma unroll
    for (int q = 0; q < R; ++q) o[b + q * B] = x[q];
  }
  if constexpr (LAST) {
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = o[e];
  } else {
    TOPT_STRESS_POINT(NS * 17 + 1);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int j = t + b * T;
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int q = 0; q < R; ++q) line[rf_idx<LS, rf_log2(E)>(base + q * NS)] = o[b + q * B];
    }
    rf_sync<WARP>();
    TOPT_STRESS_POINT(NS * 17 + 2);
#pragma unroll
    for (int e = 0; e < E; ++e) a[e] = line[rf_idx<LS, rf_log2(E)>(t + T * e)];
    rf_sync<WARP>();
    rf_stage<N, E, NS * R, OFF + (NS > 1 ? B * NB : 0), INV, WARP, FULL, LS, C>(a, line, t, tw);
  }
}

// Unnormalised DFT of the line held in a[] (forward exp(-i k x), inverse exp(+i k x)).
// `line` is this line's smem scratch (RfCfg::STRIDE complex); `tw` from rf_twiddles with the
// same FULL; every thread of the sync group (warp if WARP, else block) must call it.
template <int N, int E, bool INV, bool WARP, bool FULL = false, int LS = 0, typename C>
__device__ __forceinline__ void rf_fft(C (&a)[E], C* line, int t, const C* tw) {
  rf_stage<N, E, 1, 0, INV, WARP, FULL, LS, C>(a, line, t, tw);
}

// Two independent lines (possibly of different precisions) transformed in lock step: the same
// stage sequence as rf_stage, both lines' butterflies between one pair of barriers (half the
// barriers of two rf_fft calls, twice the independent work between them).  line1 / line2 are
// disjoint scratch lines.
template <int N, int E, int NS, int OFF, bool INV, bool WARP, bool FULL, int LS, typename C1, typename C2>
__device__ __forceinline__ void rf_stage2(C1 (&a1)[E], C1* line1, const C1* tw1, C2 (&a2)[E], C2* line2,
                                          const C2* tw2, int t) {
  constexpr int R = rf_rad(N, E, NS), B = E / R, T = N / E, NB = rf_nb(R, FULL);
  constexpr bool LAST = NS * R == N;
  C1 o1[E];
  C2 o2[E];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    C1 x1[R];
    C2 x2[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      x1[r] = a1[b + r * B];
      x2[r] = a2[b + r * B];
    }
    if constexpr (NS > 1) {
      C1 w1[R];
      C2 w2[R];
      if constexpr (FULL) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          w1[r] = tw1[OFF + b * NB + r - 1];
          w2[r] = tw2[OFF + b * NB + r - 1];
        }
      } else {
        rf_powers<R>(tw1 + OFF + b * NB, w1);
        rf_powers<R>(tw2 + OFF + b * NB, w2);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) {
        x1[r] = INV ? cmulconj(x1[r], w1[r]) : cmul(x1[r], w1[r]);
        x2[r] = INV ? cmulconj(x2[r], w2[r]) : cmul(x2[r], w2[r]);
      }
    }
    Dft<R, INV, C1>::run(x1);
    Dft<R, INV, C2>::run(x2);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      o1[b + q * B] = x1[q];
      o2[b + q * B] = x2[q];
    }
  }
  if constexpr (LAST) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a1[e] = o1[e];
      a2[e] = o2[e];
    }
  } else {
    TOPT_STRESS_POINT(NS * 17 + 3);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int j = t + b * T;
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int q = 0; q < R; ++q) {
        line1[rf_idx<LS, rf_log2(E)>(base + q * NS)] = o1[b + q * B];
        line2[rf_idx<LS, rf_log2(E)>(base + q * NS)] = o2[b + q * B];
      }
    }
    rf_sync<WARP>();
    TOPT_STRESS_POINT(NS * 17 + 4);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a1[e] = line1[rf_idx<LS, rf_log2(E)>(t + T * e)];
      a2[e] = line2[rf_idx<LS, rf_log2(E)>(t + T * e)];
    }
    rf_sync<WARP>();
    rf_stage2<N, E, NS * R, OFF + (NS > 1 ? B * NB : 0), INV, WARP, FULL, LS>(a1, line1, tw1, a2, line2, tw2, t);
  }
}
template <int N, int E, bool INV, bool WARP, bool FULL = false, int LS = 0, typename C1, typename C2>
__device__ __forceinline__ void rf_fft2(C1 (&a1)[E], C1* line1, const C1* tw1, C2 (&a2)[E], C2* line2,
                                        const C2* tw2, int t) {
  rf_stage2<N, E, 1, 0, INV, WARP, FULL, LS>(a1, line1, tw1, a2, line2, tw2, t);
}

}  // namespace topt
