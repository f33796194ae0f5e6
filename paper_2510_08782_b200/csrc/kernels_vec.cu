// kernels_vec.cu — reductions, NGMRES Gram inner products and mixing (sm_100a).
//
// PAPER.md Alg. 1 line 5 / Alg. 3 line 8: the LSQ over
// g(q) - g(v^{k-i}) is assembled on the host from fp64 inner products computed here
// in one fused pass over a and every b_i ("multi-dot"); Alg. 1 line 6 / Alg. 3
// line 9: v^{k+1} = q + sum beta_i (q - v^{k-i}) in one pass ("mix").
// All reductions use fp64 per-block partials and a fixed-order finalisation.
#include <algorithm>
#include <atomic>

#include "internal.cuh"

namespace topt {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }
void launch_count_add(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// dst = scale * (sum or max) of partials[slot * kMaxPartials + 0 .. nparts-1]
__global__ void k_finalize(const double* __restrict__ partials, int nparts, double scale, int is_max,
                           double* __restrict__ dst, size_t slot_stride) {
  const double* p = partials + blockIdx.x * slot_stride;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = is_max ? fmax(acc, p[i]) : acc + p[i];
  __shared__ double sh[1024];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = is_max ? fmax(sh[threadIdx.x], sh[threadIdx.x + s])
                                                  : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) dst[blockIdx.x] = scale * sh[0];
}

void launch_finalize(const double* partials, int slot, int nparts, double scale, bool is_max,
                     double* dst, cudaStream_t st) {
  k_finalize<<<1, 1024, 0, st>>>(partials + (size_t)slot * kMaxPartials, nparts, scale, is_max ? 1 : 0,
                                 dst, kMaxPartials);
  count_launch();
}

void launch_finalize_multi(const double* partials, int slot0, int nslots, int nparts, double scale,
                           double* dst, cudaStream_t st) {
  k_finalize<<<nslots, 1024, 0, st>>>(partials + (size_t)slot0 * nparts, nparts, scale, 0, dst,
                                      (size_t)nparts);
  count_launch();
}

__global__ void k_combine_obj(double* s) { s[TOPT_S_OBJ] = s[TOPT_S_DIST] + s[TOPT_S_REG]; }

// slots [first, first + count) -> dst[0..count), each slot of `nparts` partials (stride kMaxPartials)
__global__ void k_finalize_slots(const double* __restrict__ partials, int nparts, int first_is_max,
                                 double* __restrict__ dst) {
  const double* p = partials + (size_t)blockIdx.x * kMaxPartials;
  const bool mx = first_is_max && blockIdx.x == 0;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = mx ? fmax(acc, p[i]) : acc + p[i];
  __shared__ double sh[1024];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = mx ? fmax(sh[threadIdx.x], sh[threadIdx.x + s]) : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) dst[blockIdx.x] = sh[0];
}

// dst[i] = scale * sum of slot (first + i) (slots kMaxPartials apart), i < count
void launch_finalize_multi_k(const double* partials, int first, int count, int nparts, double scale, double* dst,
                             cudaStream_t st) {
  k_finalize<<<count, 1024, 0, st>>>(partials + (size_t)first * kMaxPartials, nparts, scale, 0, dst, kMaxPartials);
  count_launch();
}

void launch_finalize_slots(const double* partials, int first, int count, int nparts, bool first_is_max,
                           double* dst, cudaStream_t st) {
  k_finalize_slots<<<count, 1024, 0, st>>>(partials + (size_t)first * kMaxPartials, nparts, first_is_max ? 1 : 0, dst);
  count_launch();
}

// Public scalars from the internal sums (h^d = cellvol, n = points):
//   GRAD_INF = max|g|, GS = h^d sum g s, REG = h^d/2 sum v u (u = alpha L v, R23),
//   SLV = h^d sum s u (= alpha <s, L v>), SLS = alpha <s, L s> = -<s, P_0 g>_h
//       = -h^d (sum g s - sum_c (sum g_c)(sum s_c)/n)     (alpha L s = -P_0 g)
__global__ void k_finish(const double* __restrict__ isc, double* __restrict__ sc, int d, double n, double cv) {
  sc[TOPT_S_GRAD_INF] = isc[I_GMAX];
  sc[TOPT_S_GS] = cv * isc[I_GS];
  sc[TOPT_S_REG] = 0.5 * cv * isc[I_VU];
  sc[TOPT_S_SLV] = cv * isc[I_SU];
  double m = 0.0;
  for (int c = 0; c < d; ++c) m += isc[I_SUMG + c] * isc[I_SUMS + c];
  sc[TOPT_S_SLS] = -cv * (isc[I_GS] - m / n);
  sc[TOPT_S_OBJ] = sc[TOPT_S_DIST] + sc[TOPT_S_REG];
  for (int i = TOPT_S_SLS + 1; i < TOPT_NSCALARS; ++i) sc[i] = 0.0;  // reserved slots: defined zeros
}
void launch_finish(const double* isc, double* sc, int d, double n, double cellvol, cudaStream_t st) {
  k_finish<<<1, 1, 0, st>>>(isc, sc, d, n, cellvol);
  count_launch();
}
__global__ void k_flag_to_double(const int* f, double* d) { *d = (double)*f; }
void launch_flag_to_double(const int* f, double* d, cudaStream_t st) {
  k_flag_to_double<<<1, 1, 0, st>>>(f, d);
  count_launch();
}
void launch_combine_obj(double* scalars, cudaStream_t st) { k_combine_obj<<<1, 1, 0, st>>>(scalars);   count_launch();
}

// Note: products are formed in fp32 (exact for fp32 x fp32 -> fp64 only if promoted first);
// promote before multiplying so every product is exact in fp64.
template <int CH>
__global__ void __launch_bounds__(kThreads) k_multidot_exact(const float* __restrict__ a, VecList L, int i0,
                                                             int count, size_t n4,
                                                             double* __restrict__ partials) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 0.0;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 x = a4[i];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (i0 + c < count) {
        const float4 y = reinterpret_cast<const float4*>(L.p[i0 + c])[i];
        double t = (double)x.x * (double)y.x;
        t = fma((double)x.y, (double)y.y, t);
        t = fma((double)x.z, (double)y.z, t);
        t = fma((double)x.w, (double)y.w, t);
        acc[c] += t;
      }
    }
  }
  __shared__ double sh[CH][kThreads / 32];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[c][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < CH && i0 + (int)threadIdx.x < count) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += sh[threadIdx.x][w];
    partials[(size_t)(i0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

void launch_multidot(const float* a, const float* const* bs, int count, size_t n, double* partials,
                     int* nparts, cudaStream_t st) {
  VecList L;
  for (int i = 0; i < count && i < kMaxVecs; ++i) L.p[i] = bs[i];
  const size_t n4 = n / 4;
  const int nb = grid_for(n4, kThreads, 148 * 8);
  *nparts = nb;
  constexpr int CH = 8;
  for (int i0 = 0; i0 < count; i0 += CH)
  {
    k_multidot_exact<CH><<<nb, kThreads, 0, st>>>(a, L, i0, count, n4, partials);
    count_launch();
  }
}

// out = q + sum_i beta_i (q - v_i): the differences are formed first (no 1 + sum beta cancellation)
__global__ void __launch_bounds__(kThreads) k_mix(const float* __restrict__ q, VecList L, int count, size_t n4,
                                                  float* __restrict__ out) {
  const float4* q4 = reinterpret_cast<const float4*>(q);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 x = q4[i];
    float4 r = x;
    for (int c = 0; c < count; ++c) {
      const float4 y = reinterpret_cast<const float4*>(L.p[c])[i];
      const float b = L.c[c];
      r.x = fmaf(b, x.x - y.x, r.x); r.y = fmaf(b, x.y - y.y, r.y);
      r.z = fmaf(b, x.z - y.z, r.z); r.w = fmaf(b, x.w - y.w, r.w);
    }
    o4[i] = r;
  }
}

void launch_mix(const float* q, const float* const* vs, const double* beta, int count, size_t n,
                float* out, cudaStream_t st) {
  VecList L;
  for (int i = 0; i < count && i < kMaxVecs; ++i) {
    L.p[i] = vs[i];
    L.c[i] = (float)beta[i];
  }
  const size_t n4 = n / 4;
  k_mix<<<grid_for(n4, kThreads, 148 * 8), kThreads, 0, st>>>(q, L, count, n4, out);
  count_launch();
}

// out = x + a*y + cst_c (cst per component c = i / (n/ncomp); used for u_q = u - rho (g - gbar))
__global__ void k_axpy_c(const float* __restrict__ x, float a, const float* __restrict__ y, size_t n4,
                         size_t comp4, float c0, float c1, float c2, float* __restrict__ out) {
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* y4 = reinterpret_cast<const float4*>(y);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / comp4;
    const float k = c == 0 ? c0 : (c == 1 ? c1 : c2);
    const float4 u = x4[i], w = y4[i];
    o4[i] = make_float4(fmaf(a, w.x, u.x) + k, fmaf(a, w.y, u.y) + k, fmaf(a, w.z, u.z) + k, fmaf(a, w.w, u.w) + k);
  }
}
void launch_axpy_c(const float* x, float a, const float* y, size_t n, int ncomp, const float* cst, float* out,
                   cudaStream_t st) {
  k_axpy_c<<<grid_for(n / 4, kThreads, 148 * 8), kThreads, 0, st>>>(x, a, y, n / 4, n / 4 / ncomp, cst[0],
                                                                     ncomp > 1 ? cst[1] : 0.f,
                                                                     ncomp > 2 ? cst[2] : 0.f, out);
  count_launch();
}

__global__ void k_axpy(const float* __restrict__ x, float a, const float* __restrict__ y, size_t n4,
                       float* __restrict__ out) {
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* y4 = reinterpret_cast<const float4*>(y);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 u = x4[i], w = y4[i];
    o4[i] = make_float4(fmaf(a, w.x, u.x), fmaf(a, w.y, u.y), fmaf(a, w.z, u.z), fmaf(a, w.w, u.w));
  }
}
void launch_axpy(const float* x, float a, const float* y, size_t n, float* out, cudaStream_t st) {
  k_axpy<<<grid_for(n / 4, kThreads, 148 * 8), kThreads, 0, st>>>(x, a, y, n / 4, out);
  count_launch();
}

__global__ void k_sub(const float* __restrict__ a, const float* __restrict__ b, size_t n4, float* __restrict__ out) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 u = a4[i], w = b4[i];
    o4[i] = make_float4(u.x - w.x, u.y - w.y, u.z - w.z, u.w - w.w);
  }
}
void launch_sub(const float* a, const float* b, size_t n, float* out, cudaStream_t st) {
  k_sub<<<grid_for(n / 4, kThreads, 148 * 8), kThreads, 0, st>>>(a, b, n / 4, out);
  count_launch();
}


// ---- z-slab window sizing: max |x| as ordered float bits ------------------------------------
__global__ void __launch_bounds__(kThreads) k_absmax(const float* __restrict__ a, const float* __restrict__ b, size_t n,
                                                     unsigned* acc) {
  float m = 0.0f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    m = fmaxf(m, fabsf(a[i]));
    if (b) m = fmaxf(m, fabsf(b[i]));
    if (a[i] != a[i] || (b && b[i] != b[i])) m = __int_as_float(0x7f800000);  // NaN: treat as unbounded
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(acc, __float_as_uint(m));
}
__global__ void k_uint_as_float_to_double(const unsigned* acc, double* d) { *d = (double)__uint_as_float(*acc); }

void launch_absmax(const float* a, const float* b, size_t n, unsigned* acc, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((n + kThreads - 1) / kThreads, 148 * 8);
  k_absmax<<<blocks, kThreads, 0, st>>>(a, b, n, acc);
  count_launch();
}
void launch_uint_as_float_to_double(const unsigned* acc, double* d, cudaStream_t st) {
  k_uint_as_float_to_double<<<1, 1, 0, st>>>(acc, d);
  count_launch();
}

}  // namespace topt
