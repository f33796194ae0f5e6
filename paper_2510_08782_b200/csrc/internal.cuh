// internal.cuh — shared definitions of the topt library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/topt.h"

namespace topt {

constexpr int kThreads = 256;
constexpr int kMaxPartials = 1 << 17;  // per reduction slot
constexpr int kNumSlots = 16;        // reduction slots in the partials buffer

// Geometry of the (local) grid handed to kernels.  Powers of two only.
struct Geom {
  int d;            // 2 or 3
  int nx, ny, nz;   // local extents (nz = 1 for d = 2)
  int lx, ly, lz;   // log2 of extents
  size_t F;         // points per scalar field
  float cx, cy, cz; // dt / h_a  (cells per unit velocity per time step)
};

// Reduction helper: per-block fp64 partials, finalised in fixed order.
struct Reduce {
  double* partials;  // [kNumSlots][kMaxPartials]
  double* scalars;   // [TOPT_NSCALARS] (device)
};

int grid_for(size_t n, int threads = kThreads, int max_blocks = kMaxPartials);

constexpr int kMaxWeights = 64;  // n_t + 1 <= 64
struct DerivWeights { float w[kMaxWeights]; };
constexpr int kMaxVecs = 64;     // pointers per multidot / mix call
struct VecList { const float* p[kMaxVecs]; float c[kMaxVecs]; };

void upload_twiddles();

// ---- semi-Lagrangian kernels (kernels_sl.cu) --------------------------------------
void launch_trace(const Geom& g, const float* v, float* df, float* da, cudaStream_t st);
// out = I[in](l + delta) (* E if E != nullptr)
void launch_sl_step(const Geom& g, const float* in, const float* delta, const float* E, float* out,
                    cudaStream_t st);
// last forward step: mS = I[in](l+delta)(*E); lam = m1 - mS; partial sum (mS - m1)^2 -> slot
void launch_sl_last(const Geom& g, const float* in, const float* delta, const float* E,
                    const float* m1, float* mS, float* lamS, double* partials, int* nparts,
                    cudaStream_t st);
// E = 1 + sgn dt/2 (a + b) + dt^2/2 a b,  a = I[divv](l + delta), b = divv
void launch_efactor(const Geom& g, const float* divv, const float* delta, float sgn_half_dt,
                    float half_dt2, float* E, cudaStream_t st);

// ---- spectral kernels (kernels_spectral.cu) ------------------------------------------
// out = beta*out + sum_{j<J} w_j * (lam_j ? lam_j : 1) * d/dx_axis psi_j
// psi_j = psi + j*psi_stride, lam_j = lam + j*lam_stride (lam may be null).
struct DerivArgs {
  const float* psi; size_t psi_stride;
  const float* lam; size_t lam_stride;
  const double* w;  // host weights, J entries (copied into kernel args)
  int J;
  float beta;       // 0 or 1
  float* out;
};
void launch_deriv_accum(const Geom& g, int axis, const DerivArgs& a, cudaStream_t st);

// Preconditioner / projection passes on Z_c = v_c + i b_c (c < d):
//   g = alpha L v + b   (Leray if leray), s = -(alpha L~)^{-1} g
// Outputs g, s (either may be null), fp64 partials for ||g||_inf, <g,s>, and the
// spectral sums reg, <s,Lv>, <s,Ls>.
struct PrecondArgs {
  const float* v;     // d*F or null (treated as 0)
  const float* b;     // d*F or null (treated as 0)
  float2* Z;          // d*F complex workspace
  float* g;           // d*F or null
  float* s;           // d*F or null
  double alpha;
  int p;              // reg order
  bool leray;
  double* partials;   // reduction buffer
  double* scalars;    // device scalars
  double cellvol;     // h^d
};
void launch_precond(const Geom& g, const PrecondArgs& a, cudaStream_t st);

// ---- vector kernels (kernels_vec.cu) ------------------------------------------------
void launch_finalize(const double* partials, int slot, int nparts, double scale, bool is_max,
                     double* dst, cudaStream_t st);
// dst[i] = scale * sum of partials slot (slot0 + i), i < nslots
void launch_finalize_multi(const double* partials, int slot0, int nslots, int nparts, double scale,
                           double* dst, cudaStream_t st);
void launch_combine_obj(double* scalars, cudaStream_t st);  // OBJ = DIST + REG
void launch_multidot(const float* a, const float* const* bs, int count, size_t n, double* partials,
                     int* nparts, cudaStream_t st);
void launch_mix(const float* q, const float* const* vs, const double* beta, int count, size_t n,
                float* out, cudaStream_t st);
void launch_axpy(const float* x, float a, const float* y, size_t n, float* out, cudaStream_t st);  // out = x + a*y
void launch_sub(const float* a, const float* b, size_t n, float* out, cudaStream_t st);           // out = a - b

}  // namespace topt
