// api.cu — C ABI of libtopt: context, workspace, gradient evaluation and the GA-NGMRES
// driver (host logic; every field operation runs in the kernels of kernels_*.cu).
//
// PAPER.md anchors: objective (1.1a) P:25-29; reduced gradient (2.2) P:105-108;
// adjoint (2.3) P:110-121 (R1); time grid/trapezoid P:126; kernel fix P:134; SL RK2
// P:136; Armijo with memory P:152-157 (R12); RPGD/FP map (2.6)/(2.7) P:168-185;
// NGMRES Alg. 1; AA Alg. 2; GA-NGMRES Alg. 3 P:244-263 (R13-R17).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "internal.cuh"

#ifdef TOPT_WITH_NCCL
#include <nccl.h>
#endif

using namespace topt;

namespace {

thread_local std::string g_err;

topt_status fail(topt_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define TOPT_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(TOPT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

#define TOPT_CHECK_LAUNCH() TOPT_CUDA(cudaGetLastError())

bool pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(int n) { int l = 0; while ((1 << l) < n) ++l; return l; }
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

struct topt_ctx {
  topt_params p{};
  int rank = 0, world = 1, device = 0;
  Geom g{};
  int d = 3;
  int nzg = 1;  // global n[2]
  int z0 = 0;
  size_t F = 0;     // local points per scalar field
  size_t vecN = 0;  // d * F
  double h[3]{}, dt = 0, cellvol = 0;
  std::vector<double> wts;  // trapezoid weights (R10)
  // workspace
  char* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0;
  float *m_traj{}, *lam_traj{}, *df{}, *da{}, *E{}, *divv{}, *b{}, *tmp{};
  float2* Z{};
  float *m0b{}, *m1b{}, *vb{}, *vt{};
  float *vcur{}, *gcur{}, *scur{}, *q{}, *gq{}, *sq{}, *vnew{}, *gnew{}, *snew{};
  float* hist{};  // (w+1) slots x 2 vectors (NGMRES: v, g; AA: r, q)
  double* partials{};
  double* sc{};    // 4 sets of TOPT_NSCALARS: [0] current, [1] trial, [2] q, [3] new
  double* dots{};  // kMaxVecs doubles
  bool have_eval = false;
  std::vector<double> replay;
#ifdef TOPT_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
};

extern "C" {

int32_t topt_abi_version(void) { return TOPT_ABI_VERSION; }

const char* topt_last_error(void) { return g_err.c_str(); }

topt_status topt_get_unique_id(uint8_t id[128]) {
#ifdef TOPT_WITH_NCCL
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return fail(TOPT_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(id, u.internal, 128);
  return TOPT_OK;
#else
  (void)id;
  return fail(TOPT_ERR_UNSUPPORTED, "libtopt built without NCCL");
#endif
}

static topt_status validate(const topt_params* p, int world) {
  if (!p) return fail(TOPT_ERR_INVALID_ARG, "params is NULL");
  if (p->dim != 2 && p->dim != 3) return fail(TOPT_ERR_INVALID_ARG, "dim must be 2 or 3");
  for (int a = 0; a < p->dim; ++a) {
    if (p->n[a] < 4 || (p->n[a] % 2)) return fail(TOPT_ERR_INVALID_ARG, "n[i] must be even and >= 4");
    if (!pow2(p->n[a]) || p->n[a] < 8 || p->n[a] > 1024)
      return fail(TOPT_ERR_UNSUPPORTED, "n[i] must be a power of two in [8, 1024]");
  }
  if (p->dim == 2 && p->n[2] != 1) return fail(TOPT_ERR_INVALID_ARG, "dim == 2 requires n[2] == 1");
  if (p->nt < 1 || p->nt + 1 > kMaxWeights) return fail(TOPT_ERR_INVALID_ARG, "nt must be in [1, 63]");
  if (p->model < 0 || p->model > 2) return fail(TOPT_ERR_INVALID_ARG, "model");
  if (p->reg_order < 1 || p->reg_order > 3) return fail(TOPT_ERR_INVALID_ARG, "reg_order must be 1, 2 or 3");
  if (!(p->alpha > 0)) return fail(TOPT_ERR_INVALID_ARG, "alpha must be > 0");
  if (p->window < 0 || p->window + 2 > kMaxVecs) return fail(TOPT_ERR_INVALID_ARG, "window must be in [0, 62]");
  if (p->sigma < 1 || p->tau < 0) return fail(TOPT_ERR_INVALID_ARG, "need sigma >= 1 and tau >= 0");
  if (p->method != TOPT_GA_NGMRES && p->method != TOPT_GA_AA) return fail(TOPT_ERR_INVALID_ARG, "method");
  if (p->ordering != TOPT_ORDER_GA && p->ordering != TOPT_ORDER_REVERSE)
    return fail(TOPT_ERR_INVALID_ARG, "ordering");
  if (p->max_iter < 0 || !(p->eps_rel >= 0) || !(p->armijo_c > 0) || p->max_backtracks < 0)
    return fail(TOPT_ERR_INVALID_ARG, "stopping / line-search parameters");
  if (world < 1) return fail(TOPT_ERR_INVALID_ARG, "world must be >= 1");
  if (world > 1) {
    if (p->dim != 3) return fail(TOPT_ERR_INVALID_ARG, "dim == 2 runs on one rank");
    if (p->n[2] % world) return fail(TOPT_ERR_INVALID_ARG, "n[2] % world != 0");
  }
  return TOPT_OK;
}

topt_status topt_create(const topt_params* p, int32_t rank, int32_t world, const uint8_t* id,
                        int32_t device, topt_ctx** out) {
  if (!out) return fail(TOPT_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  topt_status s = validate(p, world);
  if (s != TOPT_OK) return s;
  if (rank < 0 || rank >= world) return fail(TOPT_ERR_INVALID_ARG, "rank out of range");
  if (world > 1) {
    (void)id;
    return fail(TOPT_ERR_UNSUPPORTED, "z-slab decomposition (world > 1) not built in this version");
  }
  TOPT_CUDA(cudaSetDevice(device));
  auto* c = new topt_ctx();
  c->p = *p;
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->d = p->dim;
  c->nzg = p->dim == 3 ? p->n[2] : 1;
  const int nzl = c->nzg / world;
  c->z0 = rank * nzl;
  Geom& g = c->g;
  g.d = p->dim;
  g.nx = p->n[0];
  g.ny = p->n[1];
  g.nz = nzl;
  g.lx = ilog2(g.nx);
  g.ly = ilog2(g.ny);
  g.lz = ilog2(g.nz);
  g.F = (size_t)g.nx * g.ny * g.nz;
  c->F = g.F;
  c->vecN = (size_t)c->d * g.F;
  c->dt = 1.0 / p->nt;
  c->cellvol = 1.0;
  for (int a = 0; a < c->d; ++a) {
    c->h[a] = 2.0 * M_PI / p->n[a];
    c->cellvol *= c->h[a];
  }
  g.cx = (float)(c->dt / c->h[0]);
  g.cy = (float)(c->dt / c->h[1]);
  g.cz = c->d == 3 ? (float)(c->dt / c->h[2]) : 0.f;
  c->wts.assign(p->nt + 1, c->dt);
  c->wts.front() = c->wts.back() = 0.5 * c->dt;
  // workspace size
  const size_t F = g.F, V = c->vecN, S1 = p->nt + 1, W1 = p->window + 1;
  size_t b = 0;
  auto add = [&](size_t bytes) { b += align256(bytes); };
  add(S1 * F * 4);        // m_traj
  add(S1 * F * 4);        // lam_traj
  add(V * 4); add(V * 4); // df, da
  add(F * 4); add(F * 4); // E, divv
  add(V * 4);             // b
  add(F * 4);             // tmp
  add(V * 8);             // Z (complex)
  add(F * 4); add(F * 4); add(V * 4); add(V * 4);  // m0b, m1b, vb, vt
  for (int i = 0; i < 9; ++i) add(V * 4);          // vcur..snew
  add(2 * W1 * V * 4);    // history
  add((size_t)kNumSlots * kMaxPartials * 8);
  add(4 * TOPT_NSCALARS * 8);
  add(kMaxVecs * kMaxVecs * 8);
  c->ws_need = b;
  upload_twiddles();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete c;
    return fail(TOPT_ERR_CUDA, std::string("twiddle upload: ") + cudaGetErrorString(e));
  }
  *out = c;
  return TOPT_OK;
}

topt_status topt_destroy(topt_ctx* ctx) {
  if (!ctx) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
#ifdef TOPT_WITH_NCCL
  if (ctx->comm) ncclCommDestroy(ctx->comm);
#endif
  delete ctx;
  return TOPT_OK;
}

topt_status topt_workspace_size(const topt_ctx* ctx, size_t* bytes) {
  if (!ctx || !bytes) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  *bytes = ctx->ws_need;
  return TOPT_OK;
}

topt_status topt_bind_workspace(topt_ctx* c, void* dptr, size_t bytes) {
  if (!c || !dptr) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (((uintptr_t)dptr) & 255) return fail(TOPT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (bytes < c->ws_need) return fail(TOPT_ERR_WORKSPACE, "workspace too small");
  c->ws = (char*)dptr;
  c->ws_bytes = bytes;
  const size_t F = c->F, V = c->vecN, S1 = c->p.nt + 1, W1 = c->p.window + 1;
  char* q = c->ws;
  auto take = [&](size_t bytes_) { char* r = q; q += align256(bytes_); return r; };
  c->m_traj = (float*)take(S1 * F * 4);
  c->lam_traj = (float*)take(S1 * F * 4);
  c->df = (float*)take(V * 4);
  c->da = (float*)take(V * 4);
  c->E = (float*)take(F * 4);
  c->divv = (float*)take(F * 4);
  c->b = (float*)take(V * 4);
  c->tmp = (float*)take(F * 4);
  c->Z = (float2*)take(V * 8);
  c->m0b = (float*)take(F * 4);
  c->m1b = (float*)take(F * 4);
  c->vb = (float*)take(V * 4);
  c->vt = (float*)take(V * 4);
  float** vecs[9] = {&c->vcur, &c->gcur, &c->scur, &c->q, &c->gq, &c->sq, &c->vnew, &c->gnew, &c->snew};
  for (auto pp : vecs) *pp = (float*)take(V * 4);
  c->hist = (float*)take(2 * W1 * V * 4);
  c->partials = (double*)take((size_t)kNumSlots * kMaxPartials * 8);
  c->sc = (double*)take(4 * TOPT_NSCALARS * 8);
  c->dots = (double*)take(kMaxVecs * kMaxVecs * 8);
  return TOPT_OK;
}

topt_status topt_local_slab(const topt_ctx* ctx, int32_t* z0, int32_t* nz) {
  if (!ctx || !z0 || !nz) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  *z0 = ctx->z0;
  *nz = ctx->d == 3 ? ctx->g.nz : 1;
  return TOPT_OK;
}

}  // extern "C"

// ======================================================================================
// Internal orchestration
// ======================================================================================
namespace {

topt_status need_ws(topt_ctx* c) {
  if (!c) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
  if (!c->ws) return fail(TOPT_ERR_WORKSPACE, "no workspace bound");
  return TOPT_OK;
}

bool aligned16(const void* p) { return (((uintptr_t)p) & 15) == 0; }

// div v = sum_a d_a v_a (R3), into c->divv
void compute_div(topt_ctx* c, const float* v, cudaStream_t st) {
  double one = 1.0;
  for (int a = 0; a < c->d; ++a) {
    DerivArgs da{v + a * c->F, 0, nullptr, 0, &one, 1, a == 0 ? 0.f : 1.f, c->divv};
    launch_deriv_accum(c->g, a, da, st);
  }
}

// Forward half: feet (forward, and adjoint if want_adj), static factor for the model,
// trajectory m^0..m^S (m_traj), lam^S, dist -> scalars[DIST].
void forward_half(topt_ctx* c, const float* m0, const float* m1, const float* v, bool want_adj,
                  double* scal, cudaStream_t st) {
  const Geom& g = c->g;
  const int S = c->p.nt;
  const size_t F = c->F;
  launch_trace(g, v, c->df, want_adj ? c->da : nullptr, st);
  const float* Ef = nullptr;
  if (c->p.model == TOPT_CONTINUITY) {
    compute_div(c, v, st);
    launch_efactor(g, c->divv, c->df, (float)(-0.5 * c->dt), (float)(0.5 * c->dt * c->dt), c->E, st);
    Ef = c->E;
  }
  cudaMemcpyAsync(c->m_traj, m0, F * 4, cudaMemcpyDeviceToDevice, st);
  for (int j = 0; j + 1 < S; ++j)
    launch_sl_step(g, c->m_traj + j * F, c->df, Ef, c->m_traj + (j + 1) * F, st);
  int np = 0;
  launch_sl_last(g, c->m_traj + (S - 1) * F, c->df, Ef, m1, c->m_traj + S * F, c->lam_traj + S * F,
                 c->partials, &np, st);
  launch_finalize(c->partials, 0, np, 0.5 * c->cellvol, false, scal + TOPT_S_DIST, st);
}

// Adjoint half + body force + preconditioner.  Requires forward_half(want_adj=true) or
// (want_adj=false followed by an adjoint trace, done here when need_trace).
void backward_half(topt_ctx* c, const float* v, float* gout, float* sout, double* scal, bool need_trace,
                   cudaStream_t st) {
  const Geom& g = c->g;
  const int S = c->p.nt;
  const size_t F = c->F;
  if (need_trace) launch_trace(g, v, nullptr, c->da, st);
  const float* Ea = nullptr;
  if (c->p.model == TOPT_ADVECTION) {
    compute_div(c, v, st);
    launch_efactor(g, c->divv, c->da, (float)(0.5 * c->dt), (float)(0.5 * c->dt * c->dt), c->E, st);
    Ea = c->E;
  }
  for (int j = S - 1; j >= 0; --j)
    launch_sl_step(g, c->lam_traj + (j + 1) * F, c->da, Ea, c->lam_traj + j * F, st);
  // body force (2.2) / (R8), trapezoid weights (R10)
  std::vector<double> w = c->wts;
  const bool cont = c->p.model == TOPT_CONTINUITY;
  if (cont)
    for (auto& x : w) x = -x;
  for (int a = 0; a < c->d; ++a) {
    DerivArgs da{cont ? c->lam_traj : c->m_traj, F, cont ? c->m_traj : c->lam_traj, F, w.data(), S + 1,
                 0.f, c->b + a * F};
    launch_deriv_accum(g, a, da, st);
  }
  PrecondArgs pa{v, c->b, c->Z, gout, sout, c->p.alpha, c->p.reg_order,
                 c->p.model == TOPT_INCOMPRESSIBLE, c->partials, scal, c->cellvol};
  launch_precond(g, pa, st);
  launch_combine_obj(scal, st);
}

topt_status eval_gradient(topt_ctx* c, const float* m0, const float* m1, const float* v, float* gout,
                          float* sout, double* scal, cudaStream_t st) {
  forward_half(c, m0, m1, v, true, scal, st);
  backward_half(c, v, gout, sout, scal, false, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

// Forward-only trial objective: dist (device scalar); trajectory left in m_traj.
topt_status trial_dist(topt_ctx* c, const float* m0, const float* m1, const float* v, double* scal,
                       cudaStream_t st) {
  forward_half(c, m0, m1, v, false, scal, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

// ---- small dense linear algebra on the host (fp64) --------------------------------------
// Symmetric eigen-decomposition by cyclic Jacobi (n <= 64).
void jacobi_eigen(int n, std::vector<double>& A, std::vector<double>& V, std::vector<double>& ev) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[i * n + j] * A[i * n + j];
        if (i != j) off += A[i * n + j] * A[i * n + j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = cs * akp - sn * akq;
          A[k * n + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = cs * apk - sn * aqk;
          A[q * n + k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = cs * vkp - sn * vkq;
          V[k * n + q] = sn * vkp + cs * vkq;
        }
      }
  }
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
}

// argmin_beta || r + C beta ||: G = C^T C (n x n), rhs = C^T r.  Minimum-norm solution with
// eigenvalues below 1e-12 lambda_max dropped (R15: singular values below 1e-6 sigma_max).
std::vector<double> lsq_from_gram(int n, const std::vector<double>& G, const std::vector<double>& rhs) {
  std::vector<double> A = G, V, ev;
  jacobi_eigen(n, A, V, ev);
  double lmax = 0.0;
  for (double e : ev) lmax = std::max(lmax, e);
  std::vector<double> beta(n, 0.0);
  if (!(lmax > 0.0)) return beta;
  for (int k = 0; k < n; ++k) {
    if (!(ev[k] > 1e-12 * lmax)) continue;
    double proj = 0.0;
    for (int i = 0; i < n; ++i) proj += V[i * n + k] * rhs[i];
    const double coef = -proj / ev[k];
    for (int i = 0; i < n; ++i) beta[i] += coef * V[i * n + k];
  }
  return beta;
}

struct HostScalars {
  double v[TOPT_NSCALARS];
};

topt_status fetch(topt_ctx* c, int set, HostScalars& out, cudaStream_t st) {
  TOPT_CUDA(cudaMemcpyAsync(out.v, c->sc + set * TOPT_NSCALARS, sizeof(out.v), cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

// dots[i] = <a, bs[i]> (unweighted l2 over d*F entries), returned on the host
topt_status host_dots(topt_ctx* c, const float* a, const std::vector<const float*>& bs,
                      std::vector<double>& out, cudaStream_t st) {
  out.assign(bs.size(), 0.0);
  if (bs.empty()) return TOPT_OK;
  int np = 0;
  launch_multidot(a, bs.data(), (int)bs.size(), c->vecN, c->partials, &np, st);
  launch_finalize_multi(c->partials, 0, (int)bs.size(), np, 1.0, c->dots, st);
  TOPT_CHECK_LAUNCH();
  TOPT_CUDA(cudaMemcpyAsync(out.data(), c->dots, bs.size() * 8, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ======================================================================================
// ABI entry points
// ======================================================================================
extern "C" {

topt_status topt_eval_gradient(topt_ctx* c, const float* m0, const float* m1, const float* v, float* g,
                               float* s, double* d_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (!aligned16(m0) || !aligned16(m1) || !aligned16(v) || (g && !aligned16(g)) || (s && !aligned16(s)))
    return fail(TOPT_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  return eval_gradient(c, m0, m1, v, g, s, d_scalars, st);
}

topt_status topt_eval_gradient_host(topt_ctx* c, const float* m0_h, const float* m1_h, const float* v_h,
                                    float* g_h, double* h_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0_h || !m1_h || !v_h || !h_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  TOPT_CUDA(cudaMemcpyAsync(c->m0b, m0_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(c->m1b, m1_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(c->vb, v_h, c->vecN * 4, cudaMemcpyHostToDevice, st));
  topt_status r = eval_gradient(c, c->m0b, c->m1b, c->vb, c->gcur, c->scur, c->sc, st);
  if (r != TOPT_OK) return r;
  if (g_h) TOPT_CUDA(cudaMemcpyAsync(g_h, c->gcur, c->vecN * 4, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaMemcpyAsync(h_scalars, c->sc, TOPT_NSCALARS * 8, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

topt_status topt_objective(topt_ctx* c, const float* m0, const float* m1, const float* v, double* d_scalars,
                           void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  forward_half(c, m0, m1, v, false, d_scalars, st);
  PrecondArgs pa{v, nullptr, c->Z, nullptr, nullptr, c->p.alpha, c->p.reg_order, false, c->partials,
                 c->sc + 3 * TOPT_NSCALARS, c->cellvol};
  launch_precond(c->g, pa, st);
  TOPT_CUDA(cudaMemcpyAsync(d_scalars + TOPT_S_REG, c->sc + 3 * TOPT_NSCALARS + TOPT_S_REG, 8,
                            cudaMemcpyDeviceToDevice, st));
  launch_combine_obj(d_scalars, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_feet(topt_ctx* c, const float* v, float* delta_f, float* delta_a, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!v || (!delta_f && !delta_a)) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  launch_trace(c->g, v, delta_f, delta_a, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_forward(topt_ctx* c, const float* m0, const float* v, float* m_traj, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !v || !m_traj) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  // m1 unused for the trajectory; pass m0 so lam^S/dist are well defined scratch values
  forward_half(c, m0, m0, v, false, c->sc + 3 * TOPT_NSCALARS, st);
  TOPT_CUDA(cudaMemcpyAsync(m_traj, c->m_traj, (c->p.nt + 1) * c->F * 4, cudaMemcpyDeviceToDevice, st));
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_get_adjoint(topt_ctx* c, float* lam_traj, float* body_force, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  if (lam_traj)
    TOPT_CUDA(cudaMemcpyAsync(lam_traj, c->lam_traj, (c->p.nt + 1) * c->F * 4, cudaMemcpyDeviceToDevice, st));
  if (body_force) TOPT_CUDA(cudaMemcpyAsync(body_force, c->b, c->vecN * 4, cudaMemcpyDeviceToDevice, st));
  return TOPT_OK;
}

topt_status topt_derivative(topt_ctx* c, const float* f, int32_t axis, float* out, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!f || !out) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (axis < 0 || axis >= c->d) return fail(TOPT_ERR_INVALID_ARG, "axis out of range");
  double one = 1.0;
  DerivArgs da{f, 0, nullptr, 0, &one, 1, 0.f, out};
  launch_deriv_accum(c->g, axis, da, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_apply_precond(topt_ctx* c, const float* g, float* s, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!g || !s) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  PrecondArgs pa{nullptr, g, c->Z, nullptr, s, c->p.alpha, c->p.reg_order,
                 c->p.model == TOPT_INCOMPRESSIBLE, c->partials, nullptr, c->cellvol};
  launch_precond(c->g, pa, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_leray(topt_ctx* c, const float* u, float* out, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!u || !out) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  PrecondArgs pa{nullptr, u, c->Z, out, nullptr, c->p.alpha, c->p.reg_order, true, c->partials, nullptr,
                 c->cellvol};
  launch_precond(c->g, pa, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_multidot(topt_ctx* c, const float* a, const float* const* bs, int32_t count, double* d_dots,
                          void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!a || !bs || !d_dots || count < 1 || count > kMaxVecs) return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  int np = 0;
  launch_multidot(a, bs, count, c->vecN, c->partials, &np, st);
  launch_finalize_multi(c->partials, 0, count, np, 1.0, d_dots, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_mix(topt_ctx* c, const float* q, const float* const* vs, const double* beta, int32_t count,
                     float* out, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!q || !out || count < 0 || count > kMaxVecs || (count && (!vs || !beta)))
    return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  launch_mix(q, vs, beta, count, c->vecN, out, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_set_step_replay(topt_ctx* c, const double* rho, int32_t count) {
  if (!c || count < 0 || (count && !rho)) return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  c->replay.assign(rho, rho + count);
  return TOPT_OK;
}

// GA-NGMRES(w; sigma, tau) (Alg. 3) / GA-AA, host-driven.
topt_status topt_solve(topt_ctx* c, const float* m0, const float* m1, float* v_inout, topt_report* rep,
                       void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v_inout || !rep) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const topt_params& P = c->p;
  const size_t V = c->vecN;
  const int W1 = P.window + 1;
  const bool aa = P.method == TOPT_GA_AA;
  std::memset(rep, 0, sizeof(*rep));
  const double t0 = now();
  double t_pde = 0.0, t_ls = 0.0;
  int grad_evals = 0, obj_evals = 0, nsteps = 0;
  std::deque<double> replay(c->replay.begin(), c->replay.end());

  auto slot_a = [&](int i) { return c->hist + (size_t)(2 * i) * V; };      // NGMRES: v ; AA: r
  auto slot_b = [&](int i) { return c->hist + (size_t)(2 * i + 1) * V; };  // NGMRES: g ; AA: q
  std::deque<int> win;                       // ring slots, most recent last
  std::vector<std::vector<double>> H(W1, std::vector<double>(W1, 0.0));  // <g_i, g_j> by slot

  // v^0 and g(v^0)
  TOPT_CUDA(cudaMemcpyAsync(c->vcur, v_inout, V * 4, cudaMemcpyDeviceToDevice, st));
  double te = now();
  topt_status r = eval_gradient(c, m0, m1, c->vcur, c->gcur, c->scur, c->sc, st);
  if (r != TOPT_OK) return r;
  ++grad_evals;
  HostScalars cur;
  if ((r = fetch(c, 0, cur, st)) != TOPT_OK) return r;
  t_pde += now() - te;
  const double g0 = cur.v[TOPT_S_GRAD_INF];
  rep->grad_inf0 = g0;

  auto push_ngmres = [&](const float* v, const float* g) -> topt_status {
    int slot;
    if ((int)win.size() < W1) {
      slot = (int)win.size();
    } else {
      slot = win.front();
      win.pop_front();
    }
    TOPT_CUDA(cudaMemcpyAsync(slot_a(slot), v, V * 4, cudaMemcpyDeviceToDevice, st));
    TOPT_CUDA(cudaMemcpyAsync(slot_b(slot), g, V * 4, cudaMemcpyDeviceToDevice, st));
    win.push_back(slot);
    std::vector<const float*> bs;
    for (int s2 : win) bs.push_back(slot_b(s2));
    std::vector<double> dd;
    topt_status rr = host_dots(c, slot_b(slot), bs, dd, st);
    if (rr != TOPT_OK) return rr;
    for (size_t i = 0; i < win.size(); ++i) {
      H[slot][win[i]] = dd[i];
      H[win[i]][slot] = dd[i];
    }
    return TOPT_OK;
  };
  if (!aa) {
    if ((r = push_ngmres(c->vcur, c->gcur)) != TOPT_OK) return r;
  }

  double rho = 1.0;
  int k = 0;
  int exit_code = TOPT_ITER_CAP;
  HostScalars qs, ns;
  while (true) {
    if (P.max_iter == 0) break;
    // ---- q(v^k): Armijo backtracking with memory --------------------------
    const double obj0 = cur.v[TOPT_S_OBJ], gs = cur.v[TOPT_S_GS];
    bool accepted = false;
    double rho_t = rho;
    te = now();
    if (!replay.empty()) {
      rho_t = replay.front();
      replay.pop_front();
      rho = rho_t;
      launch_axpy(c->vcur, (float)rho_t, c->scur, V, c->q, st);
      accepted = true;
    } else {
      for (int t = 0; t <= P.max_backtracks; ++t) {
        launch_axpy(c->vcur, (float)rho_t, c->scur, V, c->q, st);
        if ((r = trial_dist(c, m0, m1, c->q, c->sc + 1 * TOPT_NSCALARS, st)) != TOPT_OK) return r;
        ++obj_evals;
        HostScalars ts;
        if ((r = fetch(c, 1, ts, st)) != TOPT_OK) return r;
        const double reg_t = cur.v[TOPT_S_REG] + rho_t * cur.v[TOPT_S_SLV] +
                             0.5 * rho_t * rho_t * cur.v[TOPT_S_SLS];
        const double obj_t = ts.v[TOPT_S_DIST] + reg_t;
        if (obj_t < obj0 + rho_t * P.armijo_c * gs) {
          accepted = true;
          rho = t == 0 ? 2.0 * rho_t : rho_t;
          break;
        }
        rho_t *= 0.5;
      }
    }
    if (!accepted) {
      exit_code = TOPT_STAGNATED;
      t_pde += now() - te;
      break;
    }
    // g(q): needed by every NGMRES / FP step; AA needs it only when it takes the FP branch
    auto eval_q = [&]() -> topt_status {
      topt_status rr = eval_gradient(c, m0, m1, c->q, c->gq, c->sq, c->sc + 2 * TOPT_NSCALARS, st);
      if (rr != TOPT_OK) return rr;
      ++grad_evals;
      return fetch(c, 2, qs, st);
    };
    if (!aa) {
      if ((r = eval_q()) != TOPT_OK) return r;
    }
    t_pde += now() - te;

    const int period = P.sigma + P.tau;
    const bool fp_step = P.ordering == TOPT_ORDER_GA ? (k % period >= P.sigma) : (k % period < P.tau);
    const int wk = std::min(k, P.window);
    if (!aa) {
      if (fp_step) {
        std::swap(c->vcur, c->q);
        std::swap(c->gcur, c->gq);
        std::swap(c->scur, c->sq);
        cur = qs;
      } else {
        // LSQ (Alg. 3 line 8): columns C_i = g_q - g(v^{k-i}), i = 0..w_k (R13)
        const double tl = now();
        const int m = (int)win.size();  // == wk + 1
        (void)wk;
        std::vector<const float*> bs;
        for (int i = 0; i < m; ++i) bs.push_back(slot_b(win[m - 1 - i]));  // i = 0 -> v^k
        bs.push_back(c->gq);
        std::vector<double> rdots;
        if ((r = host_dots(c, c->gq, bs, rdots, st)) != TOPT_OK) return r;
        const double gam = rdots[m];
        std::vector<double> G(m * m), rhs(m);
        for (int i = 0; i < m; ++i) {
          const int si = win[m - 1 - i];
          rhs[i] = gam - rdots[i];
          for (int j = 0; j < m; ++j) {
            const int sj = win[m - 1 - j];
            G[i * m + j] = gam - rdots[i] - rdots[j] + H[si][sj];
          }
        }
        std::vector<double> beta = lsq_from_gram(m, G, rhs);
        t_ls += now() - tl;
        std::vector<const float*> vs;
        for (int i = 0; i < m; ++i) vs.push_back(slot_a(win[m - 1 - i]));
        launch_mix(c->q, vs.data(), beta.data(), m, V, c->vnew, st);
        te = now();
        if (P.model == TOPT_INCOMPRESSIBLE) {
          PrecondArgs pa{nullptr, c->vnew, c->Z, c->vnew, nullptr, P.alpha, P.reg_order, true, c->partials,
                         nullptr, c->cellvol};
          launch_precond(c->g, pa, st);
        }
        if ((r = eval_gradient(c, m0, m1, c->vnew, c->gnew, c->snew, c->sc + 3 * TOPT_NSCALARS, st)) != TOPT_OK)
          return r;
        ++grad_evals;
        if ((r = fetch(c, 3, ns, st)) != TOPT_OK) return r;
        t_pde += now() - te;
        std::swap(c->vcur, c->vnew);
        std::swap(c->gcur, c->gnew);
        std::swap(c->scur, c->snew);
        cur = ns;
        ++nsteps;
      }
      if ((r = push_ngmres(c->vcur, c->gcur)) != TOPT_OK) return r;
    } else {
      // AA (Alg. 2): r_k = v^k - q(v^k); history of (r, q)
      launch_sub(c->vcur, c->q, V, c->vt, st);  // r_k in vt
      const int m = std::min((int)win.size(), wk);  // i = 1..w_k
      if (!fp_step && m > 0) {
        const double tl = now();
        std::vector<const float*> bs;
        for (int i = 0; i < m; ++i) bs.push_back(slot_a(win[win.size() - 1 - i]));
        bs.push_back(c->vt);
        std::vector<double> rd;
        if ((r = host_dots(c, c->vt, bs, rd, st)) != TOPT_OK) return r;
        const double gam = rd[m];
        std::vector<double> Hm(m * m);
        // <r_i, r_j> among history entries: recompute (m <= w small)
        for (int i = 0; i < m; ++i) {
          std::vector<const float*> b2;
          for (int j = 0; j < m; ++j) b2.push_back(slot_a(win[win.size() - 1 - j]));
          std::vector<double> row;
          if ((r = host_dots(c, slot_a(win[win.size() - 1 - i]), b2, row, st)) != TOPT_OK) return r;
          for (int j = 0; j < m; ++j) Hm[i * m + j] = row[j];
        }
        std::vector<double> G(m * m), rhs(m);
        for (int i = 0; i < m; ++i) {
          rhs[i] = gam - rd[i];
          for (int j = 0; j < m; ++j) G[i * m + j] = gam - rd[i] - rd[j] + Hm[i * m + j];
        }
        std::vector<double> xi = lsq_from_gram(m, G, rhs);
        t_ls += now() - tl;
        std::vector<const float*> qsv;
        for (int i = 0; i < m; ++i) qsv.push_back(slot_b(win[win.size() - 1 - i]));
        launch_mix(c->q, qsv.data(), xi.data(), m, V, c->vnew, st);
        ++nsteps;
      } else {
        TOPT_CUDA(cudaMemcpyAsync(c->vnew, c->q, V * 4, cudaMemcpyDeviceToDevice, st));
      }
      // push (r_k, q_k)
      int slot;
      if ((int)win.size() < W1) slot = (int)win.size();
      else { slot = win.front(); win.pop_front(); }
      TOPT_CUDA(cudaMemcpyAsync(slot_a(slot), c->vt, V * 4, cudaMemcpyDeviceToDevice, st));
      TOPT_CUDA(cudaMemcpyAsync(slot_b(slot), c->q, V * 4, cudaMemcpyDeviceToDevice, st));
      win.push_back(slot);
      if (fp_step || m == 0) {
        te = now();
        if ((r = eval_q()) != TOPT_OK) return r;
        t_pde += now() - te;
        std::swap(c->vcur, c->q);
        std::swap(c->gcur, c->gq);
        std::swap(c->scur, c->sq);
        cur = qs;
      } else {
        te = now();
        if (P.model == TOPT_INCOMPRESSIBLE) {
          PrecondArgs pa{nullptr, c->vnew, c->Z, c->vnew, nullptr, P.alpha, P.reg_order, true, c->partials,
                         nullptr, c->cellvol};
          launch_precond(c->g, pa, st);
        }
        if ((r = eval_gradient(c, m0, m1, c->vnew, c->gnew, c->snew, c->sc + 3 * TOPT_NSCALARS, st)) != TOPT_OK)
          return r;
        ++grad_evals;
        if ((r = fetch(c, 3, ns, st)) != TOPT_OK) return r;
        t_pde += now() - te;
        std::swap(c->vcur, c->vnew);
        std::swap(c->gcur, c->gnew);
        std::swap(c->scur, c->snew);
        cur = ns;
      }
    }
    ++k;
    const double gi = cur.v[TOPT_S_GRAD_INF];
    if (!std::isfinite(gi) || !std::isfinite(cur.v[TOPT_S_OBJ]))
      return fail(TOPT_ERR_CUDA, "non-finite objective or gradient");
    if (gi <= P.eps_rel * g0) {
      exit_code = TOPT_CONVERGED;
      break;
    }
    if (k >= P.max_iter) {
      exit_code = TOPT_ITER_CAP;
      break;
    }
  }
  TOPT_CUDA(cudaMemcpyAsync(v_inout, c->vcur, V * 4, cudaMemcpyDeviceToDevice, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  rep->obj = cur.v[TOPT_S_OBJ];
  rep->dist = cur.v[TOPT_S_DIST];
  rep->reg = cur.v[TOPT_S_REG];
  rep->grad_inf = cur.v[TOPT_S_GRAD_INF];
  rep->rho = rho;
  rep->iters = k;
  rep->grad_evals = grad_evals;
  rep->obj_evals = obj_evals;
  rep->pde_solves = 2 * grad_evals + obj_evals;
  rep->exit = exit_code;
  rep->ngmres_steps = nsteps;
  rep->t_total = now() - t0;
  rep->t_pde = t_pde;
  rep->t_ls = t_ls;
  return TOPT_OK;
}

}  // extern "C"
