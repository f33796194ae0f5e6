// internal.cuh — shared definitions of the topt library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/topt.h"

namespace topt {

// Race stress and bounds checks (libtopt_stress.so, built with -DTOPT_STRESS): at the
// synchronisation points of the pipelined kernels a pseudo-random quarter of the warps sleeps for up
// to ~1 us, reshuffling the interleavings a missing barrier or an early refill would expose, and ring /
// window indices are checked (__trap on violation).  The release library compiles both to nothing.
#ifdef TOPT_STRESS
__device__ __forceinline__ void stress_point(unsigned salt) {
  unsigned h = (blockIdx.x * 0x9E3779B1u) ^ ((threadIdx.x >> 5) * 0x85EBCA77u) ^ (salt * 0xC2B2AE3Du) ^
               (unsigned)clock();
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep(32u + (h >> 22));
}
#define TOPT_STRESS_POINT(salt) ::topt::stress_point(salt)
#define TOPT_DEVICE_CHECK(cond) \
  do {                          \
    if (!(cond)) __trap();      \
  } while (0)
#else
#define TOPT_STRESS_POINT(salt) ((void)0)
#define TOPT_DEVICE_CHECK(cond) ((void)0)
#endif

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
  // z-slab decomposition (world > 1).  zh > 0: interpolated INPUT fields carry zh halo planes
  // on each side ([zh + nz + zh] planes, pointer = first halo plane) and z is not wrapped.
  int zh;
  // y-slab geometry of the z passes: global y offset of local row 0 and global ny (0 = local)
  int ky0, nyg;
  int* haloerr;     // device flag: set to 1 when a foot leaves the halo (zh > 0)
  // window path (zh > the stored halo): when nonzero, the z period of the global grid — the
  // window [zh + nz + zh] planes covers every periodic position (zh >= (nzw - nz + 3) / 2), so a
  // foot outside it is wrapped by multiples of nzw into it (any CFL)
  int nzw;
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
void count_launch();          // one per kernel launch (all wrappers)
long long launch_count();
void launch_count_add(long long n);  // graph replays add the kernels they contain

// ---- semi-Lagrangian kernels (kernels_sl.cu) --------------------------------------
// Feet; when vsum_partials != null also per-block sums of v_c into slots 0..d-1 (*nparts blocks)
void launch_trace(const Geom& g, const float* v, float* df, float* da, double* vsum_partials, int* nparts,
                  cudaStream_t st);
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

// flow map (R32): u_out = delta + I[u_in](l + delta) (d components, cells); det(I + J) with
// J[b][a] = d_a (h_b u_b) (d*d fields) and the physical displacement h_b u_b
void launch_flow_step(const Geom& g, const float* uin, const float* delta, float* uout, cudaStream_t st);
void launch_flow_det(const Geom& g, const float* u, const float* J, const double* h, float* ydisp, float* det,
                     cudaStream_t st);

// shared-memory z-marching variants (kernels_sl_tiled.cu), used when tiled_ok(g)
bool tiled_ok(const Geom& g);
void tiled_trace(const Geom& g, const float* v, float* df, float* da, double* vsum, int* nparts, cudaStream_t st);
void tiled_step(const Geom& g, const float* in, const float* delta, const float* E, float* out, cudaStream_t st);
void tiled_last(const Geom& g, const float* in, const float* delta, const float* E, const float* m1, float* mS,
                float* lamS, double* partials, int* nparts, cudaStream_t st);
void tiled_efactor(const Geom& g, const float* divv, const float* delta, float sh, float h2, float* E,
                   cudaStream_t st);

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
// z-slabs, P2P transport: body-force z pass on the y-slab rows of gy reading the slices of every
// rank's z-slab directly (psi[q], lam[q]: rank q's slice 0, slices `stride` apart, nzl planes of
// plane_src floats) and writing b_z into every rank's z-slab (out[q]); P <= 8
void launch_deriv_zpull(const Geom& gy, const float* const* psi, const float* const* lam, float* const* out, int P,
                        size_t psi_stride, size_t lam_stride, int nzl, size_t plane_src, const double* wts, int J,
                        cudaStream_t st);

// u = alpha L v (alpha L P_L v if leray); fp64 chain, Zv = 3 double2 fields of F
void launch_vchain(const Geom& g, const float* v, double2* Zv, float* u, double alpha, int p, bool leray,
                   cudaStream_t st);
// b-chain up to the x^-1 pass (Zb = 4 float2 fields of F); see kernels_spectral.cu
void launch_bchain(const Geom& g, const float* b, float2* Zb, double alpha, int p, bool leray, cudaStream_t st);
// chain phases (z-slab decomposition runs the last-axis pass on a y-slab geometry)
int vchain_nin(const Geom& g, bool leray);
int vchain_nout(const Geom& g);
int bchain_nin(const Geom& g, bool leray);
int bchain_nout(const Geom& g, bool leray);
void vchain_xy(const Geom& g, const float* v, double2* const* Z, bool leray, cudaStream_t st);
void vchain_last(const Geom& gz, double2* const* Z, double alpha, int p, bool leray, double n_total,
                 cudaStream_t st);
void vchain_inv(const Geom& g, double2* const* Z, float* u, cudaStream_t st);
// z-slabs, P2P transport (3D, non-Leray): the last-axis passes in place on the distributed
// z-slabs; tab[f * P + q] = rank q's field f, nzl planes per rank of plane_src elements
void vchain_last_remote(const Geom& gy, const void* const* tab, int P, int nzl, size_t plane_src, double alpha, int p,
                        double n_total, cudaStream_t st);
void bchain_last_remote(const Geom& gy, const void* const* tab, int P, int nzl, size_t plane_src, double alpha, int p,
                        double n_total, cudaStream_t st);
void bchain_xy(const Geom& g, const float* b, float2* const* Z, bool leray, cudaStream_t st);
void bchain_last(const Geom& gz, float2* const* Z, double alpha, int p, bool leray, double n_total,
                 cudaStream_t st);
void bchain_yinv(const Geom& g, float2* const* Z, bool leray, cudaStream_t st);
// merged chain (non-Leray): fp64 v spectra + fp32 b spectra -> g^, p^ (fp32), y^-1 of both
// (partial slots 10, 11: sum_x v.u and sum_x s.u by Parseval, *nparts blocks)
void gchain_last(const Geom& gz, double2* const* Zv, float2* const* Zb, double alpha, int p, double n_total,
                 double* partials, int* nparts, cudaStream_t st);
void gchain_yinv(const Geom& g, float2* const* Z, cudaStream_t st);
// x^-1 of the b-chain and pointwise assembly g = u + b_L, s = -(v - vbar) + p, with
// partial sums in slots 0..9 (max|g|, sum gs, sum vu, sum su, sum g_c (3), sum s_c (3)).
void launch_assemble(const Geom& g, const float2* Zb, bool leray, const float* b, const float* u, const float* v,
                     const double* vsum, float* gout, float* sout, double* partials, int* nparts, cudaStream_t st,
                     double ntot = 0.0);

// Internal scalars (per evaluation, device): sums used to finish the public scalars.
enum { I_SUMV = 0, I_GMAX = 3, I_GS = 4, I_VU = 5, I_SU = 6, I_SUMG = 7, I_SUMS = 10, I_COUNT = 16 };

// ---- vector kernels (kernels_vec.cu) ------------------------------------------------
void launch_finalize(const double* partials, int slot, int nparts, double scale, bool is_max,
                     double* dst, cudaStream_t st);
// dst[i] = scale * sum of partials slot (slot0 + i), i < nslots
void launch_finalize_multi(const double* partials, int slot0, int nslots, int nparts, double scale,
                           double* dst, cudaStream_t st);
void launch_combine_obj(double* scalars, cudaStream_t st);  // OBJ = DIST + REG
void launch_flag_to_double(const int* f, double* d, cudaStream_t st);
void launch_finalize_multi_k(const double* partials, int first, int count, int nparts, double scale, double* dst,
                             cudaStream_t st);
// finalize slots [first, first+count) (slot 0 of the assembly = max) into dst
void launch_finalize_slots(const double* partials, int first, int count, int nparts, bool first_is_max,
                           double* dst, cudaStream_t st);
// public scalars from the internal sums (see kernels_vec.cu)
void launch_finish(const double* isc, double* sc, int d, double n, double cellvol, cudaStream_t st);
void launch_multidot(const float* a, const float* const* bs, int count, size_t n, double* partials,
                     int* nparts, cudaStream_t st);
void launch_mix(const float* q, const float* const* vs, const double* beta, int count, size_t n,
                float* out, cudaStream_t st);
// *acc = max(*acc, bits of max |x|) over x = a[0..n) and b[0..n) (b may be null); non-negative floats
// order like their bit patterns, so the running maximum is an atomicMax on unsigned (caller zeroes it)
void launch_absmax(const float* a, const float* b, size_t n, unsigned* acc, cudaStream_t st);
void launch_uint_as_float_to_double(const unsigned* acc, double* d, cudaStream_t st);
void launch_axpy(const float* x, float a, const float* y, size_t n, float* out, cudaStream_t st);  // out = x + a*y
void launch_sub(const float* a, const float* b, size_t n, float* out, cudaStream_t st);           // out = a - b
void launch_axpy_c(const float* x, float a, const float* y, size_t n, int ncomp, const float* cst, float* out,
                   cudaStream_t st);  // out = x + a*y + cst[component]

}  // namespace topt
