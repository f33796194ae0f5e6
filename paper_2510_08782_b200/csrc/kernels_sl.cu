// kernels_sl.cu — semi-Lagrangian trace and step kernels (sm_100a).
//
// "semi-Lagrangian scheme ... unconditionally stable; explicit,
// second-order Runge-Kutta".  Readings:
//   R5  periodic tricubic Lagrange interpolation at node + displacement (cells);
//       the foot is kept as an fp32 displacement so the integer node index is exact
//   R6  midpoint RK2 feet: X = x - dt v(x - dt/2 v(x)), Y = x + dt v(x + dt/2 v(x))
//   R7  Heun source factor E for the conservative forms (continuity forward,
//       advection adjoint)
// The dist term of (1.1a) is fused into the last forward step with an fp64
// per-block partial sum (fixed-order finalisation => reproducible).
#include "internal.cuh"

namespace topt {

__device__ __forceinline__ void lagrange4(float t, float w[4]) {
  // nodes -1, 0, 1, 2 (R5)
  const float tm1 = t - 1.0f, tm2 = t - 2.0f, tp1 = t + 1.0f;
  w[0] = -t * tm1 * tm2 * (1.0f / 6.0f);
  w[1] = tp1 * tm1 * tm2 * 0.5f;
  w[2] = -tp1 * t * tm2 * 0.5f;
  w[3] = tp1 * t * tm1 * (1.0f / 6.0f);
}

// Stencil of one point: periodic row offsets and weights.
template <int D>
struct Stencil {
  int xo[4];          // x indices (already wrapped)
  size_t ro[D == 3 ? 16 : 4];  // row base offsets (y, z combined, wrapped)
  float wx[4], wr[D == 3 ? 16 : 4];

  __device__ __forceinline__ void build(const Geom& g, int x, int y, int z, float dx, float dy, float dz) {
    const float fx = floorf(dx), fy = floorf(dy);
    const int ix = x + (int)fx, iy = y + (int)fy;
    float wy[4];
    lagrange4(dx - fx, wx);
    lagrange4(dy - fy, wy);
#pragma unroll
    for (int a = 0; a < 4; ++a) xo[a] = (ix - 1 + a) & (g.nx - 1);
    if (D == 3) {
      const float fz = floorf(dz);
      const int iz = z + (int)fz;
      float wz[4];
      lagrange4(dz - fz, wz);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const size_t zb = (size_t)((iz - 1 + c) & (g.nz - 1)) << (g.lx + g.ly);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          ro[c * 4 + b] = zb + ((size_t)((iy - 1 + b) & (g.ny - 1)) << g.lx);
          wr[c * 4 + b] = wz[c] * wy[b];
        }
      }
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        ro[b] = (size_t)((iy - 1 + b) & (g.ny - 1)) << g.lx;
        wr[b] = wy[b];
      }
    }
  }

  __device__ __forceinline__ float apply(const float* __restrict__ f) const {
    constexpr int NR = D == 3 ? 16 : 4;
    float acc = 0.0f;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float* row = f + ro[r];
      float s = wx[0] * __ldg(row + xo[0]);
      s = fmaf(wx[1], __ldg(row + xo[1]), s);
      s = fmaf(wx[2], __ldg(row + xo[2]), s);
      s = fmaf(wx[3], __ldg(row + xo[3]), s);
      acc = fmaf(wr[r], s, acc);
    }
    return acc;
  }
};

__device__ __forceinline__ void coords(const Geom& g, size_t i, int& x, int& y, int& z) {
  x = (int)(i & (g.nx - 1));
  y = (int)((i >> g.lx) & (g.ny - 1));
  z = (int)(i >> (g.lx + g.ly));
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[w];
  return r;  // valid on thread 0
}

// K1: midpoint-RK2 feet (R6), in cells.  delta_f = -c I[v](l - c v/2), delta_a = +c I[v](l + c v/2)
// Optionally per-block sums of v_c (fp64) into partials[c * kMaxPartials + block].
template <int D>
__global__ void __launch_bounds__(kThreads) k_trace(Geom g, const float* __restrict__ v,
                                                    float* __restrict__ df, float* __restrict__ da,
                                                    double* __restrict__ vsum) {
  const size_t F = g.F;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, i, x, y, z);
    const float w0 = v[i], w1 = v[F + i], w2 = D == 3 ? v[2 * F + i] : 0.0f;
    s0 += w0; s1 += w1; s2 += w2;
    const float u0 = w0 * g.cx, u1 = w1 * g.cy, u2 = w2 * g.cz;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      float* out = side == 0 ? df : da;
      if (out == nullptr) continue;
      const float sg = side == 0 ? -1.0f : 1.0f;
      Stencil<D> st;
      st.build(g, x, y, z, 0.5f * sg * u0, 0.5f * sg * u1, 0.5f * sg * u2);
      out[i] = sg * g.cx * st.apply(v);
      out[F + i] = sg * g.cy * st.apply(v + F);
      if (D == 3) out[2 * F + i] = sg * g.cz * st.apply(v + 2 * F);
    }
  }
  if (vsum) {
    const double a = block_sum(s0);
    const double b = block_sum(s1);
    const double c = block_sum(s2);
    if (threadIdx.x == 0) {
      vsum[blockIdx.x] = a;
      vsum[kMaxPartials + blockIdx.x] = b;
      vsum[2 * kMaxPartials + blockIdx.x] = c;
    }
  }
}

// K2: one SL step  out(l) = I[in](l + delta(l)) (* E(l))
template <int D, bool HAS_E>
__global__ void __launch_bounds__(kThreads) k_sl_step(Geom g, const float* __restrict__ in,
                                                      const float* __restrict__ delta,
                                                      const float* __restrict__ E,
                                                      float* __restrict__ out) {
  const size_t F = g.F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, i, x, y, z);
    Stencil<D> st;
    st.build(g, x, y, z, delta[i], delta[F + i], D == 3 ? delta[2 * F + i] : 0.0f);
    float r = st.apply(in);
    if (HAS_E) r *= E[i];
    out[i] = r;
  }
}

// K3: last forward step + mismatch: mS, lamS = m1 - mS (R1), partial sum (mS - m1)^2
template <int D, bool HAS_E>
__global__ void __launch_bounds__(kThreads) k_sl_last(Geom g, const float* __restrict__ in,
                                                      const float* __restrict__ delta,
                                                      const float* __restrict__ E,
                                                      const float* __restrict__ m1,
                                                      float* __restrict__ mS, float* __restrict__ lamS,
                                                      double* __restrict__ partials) {
  const size_t F = g.F;
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, i, x, y, z);
    Stencil<D> st;
    st.build(g, x, y, z, delta[i], delta[F + i], D == 3 ? delta[2 * F + i] : 0.0f);
    float r = st.apply(in);
    if (HAS_E) r *= E[i];
    const float res = m1[i] - r;
    mS[i] = r;
    if (lamS) lamS[i] = res;
    acc += (double)res * (double)res;
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Static Heun factor (R7): E = 1 + sgn dt/2 (a + b) + dt^2/2 a b, a = I[divv](l+delta), b = divv(l)
template <int D>
__global__ void __launch_bounds__(kThreads) k_efactor(Geom g, const float* __restrict__ divv,
                                                      const float* __restrict__ delta, float sh,
                                                      float h2, float* __restrict__ E) {
  const size_t F = g.F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, i, x, y, z);
    Stencil<D> st;
    st.build(g, x, y, z, delta[i], delta[F + i], D == 3 ? delta[2 * F + i] : 0.0f);
    const float a = st.apply(divv), b = divv[i];
    E[i] = 1.0f + sh * (a + b) + h2 * a * b;
  }
}

// Flow map (R32): one composition step of the backward map, all d displacement components
// with one stencil: u_out_c(l) = delta_c(l) + I[u_in_c](l + delta(l))  (cells).
template <int D>
__global__ void __launch_bounds__(kThreads) k_flow_step(Geom g, const float* __restrict__ uin,
                                                        const float* __restrict__ delta,
                                                        float* __restrict__ uout) {
  const size_t F = g.F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, i, x, y, z);
    const float d0 = delta[i], d1 = delta[F + i], d2 = D == 3 ? delta[2 * F + i] : 0.0f;
    Stencil<D> st;
    st.build(g, x, y, z, d0, d1, d2);
    uout[i] = d0 + st.apply(uin);
    uout[F + i] = d1 + st.apply(uin + F);
    if (D == 3) uout[2 * F + i] = d2 + st.apply(uin + 2 * F);
  }
}

// det(I + J) with J[b][a] = d/dx_a (h_b u_b) given as d*d fields (row b, column a);
// also writes the physical displacement y_b - x_b = h_b u_b.
template <int D>
__global__ void __launch_bounds__(kThreads) k_flow_det(Geom g, const float* __restrict__ u,
                                                       const float* __restrict__ J, float hx, float hy,
                                                       float hz, float* __restrict__ ydisp,
                                                       float* __restrict__ det) {
  const size_t F = g.F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < F; i += (size_t)gridDim.x * blockDim.x) {
    if (D == 2) {
      const double a = 1.0 + J[i], b = J[F + i], c = J[2 * F + i], e = 1.0 + J[3 * F + i];
      det[i] = (float)(a * e - b * c);
      ydisp[i] = hx * u[i];
      ydisp[F + i] = hy * u[F + i];
    } else {
      double m[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) m[r][q] = (r == q ? 1.0 : 0.0) + J[(size_t)(3 * r + q) * F + i];
      det[i] = (float)(m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                       m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                       m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]));
      ydisp[i] = hx * u[i];
      ydisp[F + i] = hy * u[F + i];
      ydisp[2 * F + i] = hz * u[2 * F + i];
    }
  }
}

void launch_flow_step(const Geom& g, const float* uin, const float* delta, float* uout, cudaStream_t st);
void launch_flow_det(const Geom& g, const float* u, const float* J, const double* h, float* ydisp, float* det,
                     cudaStream_t st);

int grid_for(size_t n, int threads, int max_blocks) {
  size_t b = (n + threads - 1) / threads;
  if (b > (size_t)max_blocks) b = max_blocks;
  if (b < 1) b = 1;
  return (int)b;
}

static int sl_grid(const Geom& g) { return grid_for(g.F, kThreads, 148 * 16); }

void launch_trace(const Geom& g, const float* v, float* df, float* da, double* vsum_partials, int* nparts,
                  cudaStream_t st) {
  if (tiled_ok(g)) {
    tiled_trace(g, v, df, da, vsum_partials, nparts, st);
    return;
  }
  const int gr = sl_grid(g);
  if (nparts) *nparts = gr;
  if (g.d == 3) k_trace<3><<<gr, kThreads, 0, st>>>(g, v, df, da, vsum_partials);
  else k_trace<2><<<gr, kThreads, 0, st>>>(g, v, df, da, vsum_partials);
  count_launch();
}

void launch_sl_step(const Geom& g, const float* in, const float* delta, const float* E, float* out,
                    cudaStream_t st) {
  if (tiled_ok(g)) {
    tiled_step(g, in, delta, E, out, st);
    return;
  }
  const int gr = sl_grid(g);
  if (g.d == 3) {
    if (E) k_sl_step<3, true><<<gr, kThreads, 0, st>>>(g, in, delta, E, out);
    else k_sl_step<3, false><<<gr, kThreads, 0, st>>>(g, in, delta, E, out);
  } else {
    if (E) k_sl_step<2, true><<<gr, kThreads, 0, st>>>(g, in, delta, E, out);
    else k_sl_step<2, false><<<gr, kThreads, 0, st>>>(g, in, delta, E, out);
  }
  count_launch();
}

void launch_sl_last(const Geom& g, const float* in, const float* delta, const float* E,
                    const float* m1, float* mS, float* lamS, double* partials, int* nparts,
                    cudaStream_t st) {
  if (tiled_ok(g)) {
    tiled_last(g, in, delta, E, m1, mS, lamS, partials, nparts, st);
    return;
  }
  const int gr = grid_for(g.F, kThreads, kMaxPartials);
  *nparts = gr;
  if (g.d == 3) {
    if (E) k_sl_last<3, true><<<gr, kThreads, 0, st>>>(g, in, delta, E, m1, mS, lamS, partials);
    else k_sl_last<3, false><<<gr, kThreads, 0, st>>>(g, in, delta, E, m1, mS, lamS, partials);
  } else {
    if (E) k_sl_last<2, true><<<gr, kThreads, 0, st>>>(g, in, delta, E, m1, mS, lamS, partials);
    else k_sl_last<2, false><<<gr, kThreads, 0, st>>>(g, in, delta, E, m1, mS, lamS, partials);
  }
  count_launch();
}

void launch_flow_step(const Geom& g, const float* uin, const float* delta, float* uout, cudaStream_t st) {
  if (g.d == 3) k_flow_step<3><<<sl_grid(g), kThreads, 0, st>>>(g, uin, delta, uout);
  else k_flow_step<2><<<sl_grid(g), kThreads, 0, st>>>(g, uin, delta, uout);
  count_launch();
}

void launch_flow_det(const Geom& g, const float* u, const float* J, const double* h, float* ydisp, float* det,
                     cudaStream_t st) {
  if (g.d == 3)
    k_flow_det<3><<<sl_grid(g), kThreads, 0, st>>>(g, u, J, (float)h[0], (float)h[1], (float)h[2], ydisp, det);
  else
    k_flow_det<2><<<sl_grid(g), kThreads, 0, st>>>(g, u, J, (float)h[0], (float)h[1], 0.f, ydisp, det);
  count_launch();
}

void launch_efactor(const Geom& g, const float* divv, const float* delta, float sgn_half_dt,
                    float half_dt2, float* E, cudaStream_t st) {
  if (tiled_ok(g)) {
    tiled_efactor(g, divv, delta, sgn_half_dt, half_dt2, E, st);
    return;
  }
  if (g.d == 3) k_efactor<3><<<sl_grid(g), kThreads, 0, st>>>(g, divv, delta, sgn_half_dt, half_dt2, E);
  else k_efactor<2><<<sl_grid(g), kThreads, 0, st>>>(g, divv, delta, sgn_half_dt, half_dt2, E);
  count_launch();
}

}  // namespace topt
