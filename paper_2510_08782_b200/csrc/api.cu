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
  float *m_traj{}, *lam_traj{}, *df{}, *da{}, *E{}, *divv{}, *b{}, *utmp{};
  float2* Z{};      // b-chain: 4 complex fields of F
  double2* Zv{};    // v-chain: 3 double-complex fields of F
  float *m0b{}, *m1b{}, *vb{}, *vt{};
  float *vcur{}, *gcur{}, *scur{}, *q{}, *gq{}, *sq{}, *vnew{}, *gnew{}, *snew{};
  float *ucur{}, *uq{}, *unew{};  // u = alpha L v tracked alongside v
  float* hist{};  // (w+1) slots x 3 vectors (NGMRES: v, g, u; AA: r, q, u(q))
  double* partials{};
  double* sc{};    // 5 sets of 32: [0..15] public, [16..31] internal; sets: current, trial, q, new, scratch
  double* dots{};  // kMaxVecs doubles
  bool have_eval = false;
  std::vector<double> replay;
  // per-kernel-class timing (topt_profile / topt_kernel_stats)
  bool prof = false;
  struct Rec { int cls; cudaEvent_t a, b; double bytes; int launches; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double pms[16]{}, pbytes[16]{};
  long long plaunch[16]{};
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
  add(V * 4);             // utmp
  add(4 * F * 8);         // Z (4 complex fields)
  add(3 * F * 16);        // Zv (3 double-complex fields)
  add(F * 4); add(F * 4); add(V * 4); add(V * 4);  // m0b, m1b, vb, vt
  for (int i = 0; i < 12; ++i) add(V * 4);         // vcur..snew, ucur, uq, unew
  add(3 * W1 * V * 4);    // history
  add((size_t)kNumSlots * kMaxPartials * 8);
  add(5 * 32 * 8);
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
  for (auto& r : ctx->recs) { ctx->pool.push_back(r.a); ctx->pool.push_back(r.b); }
  for (auto e : ctx->pool) cudaEventDestroy(e);
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
  c->utmp = (float*)take(V * 4);
  c->Z = (float2*)take(4 * F * 8);
  c->Zv = (double2*)take(3 * F * 16);
  c->m0b = (float*)take(F * 4);
  c->m1b = (float*)take(F * 4);
  c->vb = (float*)take(V * 4);
  c->vt = (float*)take(V * 4);
  float** vecs[12] = {&c->vcur, &c->gcur, &c->scur, &c->q,    &c->gq,   &c->sq,
                      &c->vnew, &c->gnew, &c->snew, &c->ucur, &c->uq,   &c->unew};
  for (auto pp : vecs) *pp = (float*)take(V * 4);
  c->hist = (float*)take(3 * W1 * V * 4);
  c->partials = (double*)take((size_t)kNumSlots * kMaxPartials * 8);
  c->sc = (double*)take(5 * 32 * 8);
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

constexpr int kSet = 32;  // doubles per scalar set: [0, 16) public, [16, 32) internal

// Kernel classes for topt_kernel_stats; bytes are ALGORITHMIC (each operand read once,
// each result written once per launch group).
// K_SL_STEP: every interior SL step of both sweeps (one kernel, forward with/without E and
// adjoint); the last forward step (fused mismatch) is its own class.
enum KClass { K_TRACE, K_SL_STEP, K_SL_LAST, K_EFACTOR, K_DIV, K_BODY, K_VCHAIN, K_BCHAIN, K_ASSEMBLE, K_MISC,
              K_NCLASS };
const char* kClassNames[K_NCLASS] = {"sl_trace", "sl_step",        "sl_step_last", "efactor",  "div_v",
                                     "body_force", "vchain_alphaLv", "bchain_fft",   "assemble", "misc"};

cudaEvent_t take_event(topt_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII scope: when profiling, brackets the enclosed launches with events on `st`
struct Prof {
  topt_ctx* c;
  int cls;
  double bytes;
  int nl;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Prof(topt_ctx* c_, int cls_, double bytes_, int nl_, cudaStream_t st_)
      : c(c_), cls(cls_), bytes(bytes_), nl(nl_), st(st_) {
    if (c->prof) {
      a = take_event(c);
      cudaEventRecord(a, st);
    }
  }
  ~Prof() {
    if (c->prof) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, st);
      c->recs.push_back({cls, a, b, bytes, nl});
    }
  }
};

topt_status need_ws(topt_ctx* c) {
  if (!c) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
  if (!c->ws) return fail(TOPT_ERR_WORKSPACE, "no workspace bound");
  return TOPT_OK;
}

bool aligned16(const void* p) { return (((uintptr_t)p) & 15) == 0; }

double* pub(topt_ctx* c, int set) { return c->sc + set * kSet; }
double* intl(topt_ctx* c, int set) { return c->sc + set * kSet + 16; }

// div v = sum_a d_a v_a (R3), into c->divv
void compute_div(topt_ctx* c, const float* v, cudaStream_t st) {
  double one = 1.0;
  for (int a = 0; a < c->d; ++a) {
    DerivArgs da{v + a * c->F, 0, nullptr, 0, &one, 1, a == 0 ? 0.f : 1.f, c->divv};
    launch_deriv_accum(c->g, a, da, st);
  }
}

// Forward half: feet (R6), static factor (continuity, R7), m^0..m^S in m_traj,
// lam^S = m1 - m^S (R1/R8), dist -> scal[DIST], sum_x v_c -> isc[I_SUMV..].
void forward_half(topt_ctx* c, const float* m0, const float* m1, const float* v, bool want_adj, double* scal,
                  double* isc, cudaStream_t st) {
  const Geom& g = c->g;
  const int S = c->p.nt;
  const size_t F = c->F;
  const double F4 = 4.0 * F, d = c->d;
  int np = 0;
  {
    Prof pr(c, K_TRACE, (d + d * (want_adj ? 2 : 1)) * F4, 1, st);
    launch_trace(g, v, c->df, want_adj ? c->da : nullptr, c->partials, &np, st);
  }
  {
    Prof pr(c, K_MISC, 0.0, 1, st);
    launch_finalize_slots(c->partials, 0, c->d, np, false, isc + I_SUMV, st);
  }
  const float* Ef = nullptr;
  if (c->p.model == TOPT_CONTINUITY) {
    {
      Prof pr(c, K_DIV, (3.0 * d - 1.0) * F4, c->d, st);
      compute_div(c, v, st);
    }
    Prof pr(c, K_EFACTOR, (d + 2) * F4, 1, st);
    launch_efactor(g, c->divv, c->df, (float)(-0.5 * c->dt), (float)(0.5 * c->dt * c->dt), c->E, st);
    Ef = c->E;
  }
  const double e = Ef ? 1.0 : 0.0;
  {
    Prof pr(c, K_MISC, 2.0 * F4, 0, st);
    cudaMemcpyAsync(c->m_traj, m0, F * 4, cudaMemcpyDeviceToDevice, st);
  }
  for (int j = 0; j + 1 < S; ++j) {
    Prof pr(c, K_SL_STEP, (d + 2 + e) * F4, 1, st);
    launch_sl_step(g, c->m_traj + j * F, c->df, Ef, c->m_traj + (j + 1) * F, st);
  }
  {
    Prof pr(c, K_SL_LAST, (d + 4 + e) * F4, 1, st);
    launch_sl_last(g, c->m_traj + (S - 1) * F, c->df, Ef, m1, c->m_traj + S * F, c->lam_traj + S * F, c->partials,
                   &np, st);
  }
  Prof pr(c, K_MISC, 0.0, 1, st);
  launch_finalize(c->partials, 0, np, 0.5 * c->cellvol, false, scal + TOPT_S_DIST, st);
}

// Backward half: adjoint sweep (advection: Heun factor, R7), body force (2.2)/(R8) with
// trapezoid weights (R10), then g = alpha L v + b (P_L b for incompressible, R9) and
// s = -(alpha L~)^{-1} g = -P_0 v - (alpha L~)^{-1} b.  alpha L v is `u` when the
// caller tracks it (solver), otherwise computed by the fp64 v-chain.
void backward_half(topt_ctx* c, const float* v, const float* u, float* gout, float* sout, double* scal,
                   double* isc, cudaStream_t st) {
  const Geom& g = c->g;
  const int S = c->p.nt;
  const size_t F = c->F;
  const double F4 = 4.0 * F, d = c->d;
  const float* Ea = nullptr;
  if (c->p.model == TOPT_ADVECTION) {
    {
      Prof pr(c, K_DIV, (3.0 * d - 1.0) * F4, c->d, st);
      compute_div(c, v, st);
    }
    Prof pr(c, K_EFACTOR, (d + 2) * F4, 1, st);
    launch_efactor(g, c->divv, c->da, (float)(0.5 * c->dt), (float)(0.5 * c->dt * c->dt), c->E, st);
    Ea = c->E;
  }
  const double e = Ea ? 1.0 : 0.0;
  for (int j = S - 1; j >= 0; --j) {
    Prof pr(c, K_SL_STEP, (d + 2 + e) * F4, 1, st);
    launch_sl_step(g, c->lam_traj + (j + 1) * F, c->da, Ea, c->lam_traj + j * F, st);
  }
  std::vector<double> w = c->wts;
  const bool cont = c->p.model == TOPT_CONTINUITY;
  if (cont)
    for (auto& x : w) x = -x;
  for (int a = 0; a < c->d; ++a) {
    Prof pr(c, K_BODY, (2.0 * (S + 1) + 1.0) * F4, 1, st);
    DerivArgs da{cont ? c->lam_traj : c->m_traj, F, cont ? c->m_traj : c->lam_traj, F, w.data(), S + 1, 0.f,
                 c->b + a * F};
    launch_deriv_accum(g, a, da, st);
  }
  const bool leray = c->p.model == TOPT_INCOMPRESSIBLE;
  const double half = c->d == 3 ? 2.0 : 1.0;
  if (!u) {
    const double nin = leray ? d : half, nout = half, F16 = 16.0 * F;
    const double bytes = d * F4 + nin * F16 + (c->d == 3 ? 2 * nin * F16 + 2 * nout * F16 : 0.0) +
                         (nin + nout) * F16 + nout * F16 + d * F4;
    Prof pr(c, K_VCHAIN, bytes, c->d == 3 ? 5 : 3, st);
    launch_vchain(g, v, c->Zv, c->utmp, c->p.alpha, c->p.reg_order, leray, st);
    u = c->utmp;
  }
  {
    const double nin = leray ? d : half, nout = leray ? 2 * half : half, F8 = 8.0 * F;
    const double bytes = d * F4 + nin * F8 + (c->d == 3 ? 2 * nin * F8 + 2 * nout * F8 : 0.0) + (nin + nout) * F8;
    Prof pr(c, K_BCHAIN, bytes, c->d == 3 ? 4 : 2, st);
    launch_bchain(g, c->b, c->Z, c->p.alpha, c->p.reg_order, leray, st);
  }
  int np = 0;
  {
    const double nout = leray ? 2 * half : half;
    const double bytes = nout * 8.0 * F + (leray ? 0.0 : d * F4) + 2 * d * F4 + 2 * d * F4;
    Prof pr(c, K_ASSEMBLE, bytes, 1, st);
    launch_assemble(g, c->Z, leray, c->b, u, v, isc + I_SUMV, gout, sout, c->partials, &np, st);
  }
  Prof pr(c, K_MISC, 0.0, 2, st);
  launch_finalize_slots(c->partials, 0, 10, np, true, isc + I_GMAX, st);
  launch_finish(isc, scal, c->d, (double)F, c->cellvol, st);
}

topt_status eval_gradient(topt_ctx* c, const float* m0, const float* m1, const float* v, const float* u,
                          float* gout, float* sout, double* scal, double* isc, cudaStream_t st) {
  forward_half(c, m0, m1, v, true, scal, isc, st);
  backward_half(c, v, u, gout, sout, scal, isc, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

// Forward-only trial objective (the Armijo trial): scal[DIST].
topt_status trial_dist(topt_ctx* c, const float* m0, const float* m1, const float* v, double* scal, double* isc,
                       cudaStream_t st) {
  forward_half(c, m0, m1, v, false, scal, isc, st);
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
    if (off == 0.0 || off <= 1e-30 * tot) break;
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

// argmin_beta || r + C beta ||_2 from G = C^T C and rhs = C^T r: minimum-norm solution with
// eigenvalues of G below 1e-12 lambda_max dropped (R15: singular values of C below 1e-6 sigma_max).
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
  double v[kSet];
  double pub(int i) const { return v[i]; }
  double in(int i) const { return v[16 + i]; }
};

topt_status fetch(topt_ctx* c, int set, HostScalars& out, cudaStream_t st) {
  TOPT_CUDA(cudaMemcpyAsync(out.v, c->sc + set * kSet, sizeof(out.v), cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

// dots[i] = <a, bs[i]> (unweighted l2 over d*F entries), returned on the host
topt_status host_dots(topt_ctx* c, const float* a, const std::vector<const float*>& bs, std::vector<double>& out,
                      cudaStream_t st) {
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

// in-place Leray projection of a vector field (b-chain with b := x, assemble writes P_L x)
void leray_inplace(topt_ctx* c, float* x, cudaStream_t st) {
  launch_bchain(c->g, x, c->Z, c->p.alpha, c->p.reg_order, true, st);
  int np = 0;
  launch_assemble(c->g, c->Z, true, nullptr, nullptr, nullptr, nullptr, x, nullptr, c->partials, &np, st);
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ======================================================================================
// ABI entry points
// ======================================================================================
extern "C" {

topt_status topt_eval_gradient(topt_ctx* c, const float* m0, const float* m1, const float* v, float* g, float* s,
                               double* d_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (!aligned16(m0) || !aligned16(m1) || !aligned16(v) || (g && !aligned16(g)) || (s && !aligned16(s)))
    return fail(TOPT_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  return eval_gradient(c, m0, m1, v, nullptr, g, s, d_scalars, intl(c, 4), (cudaStream_t)stream);
}

topt_status topt_eval_gradient_host(topt_ctx* c, const float* m0_h, const float* m1_h, const float* v_h, float* g_h,
                                    double* h_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0_h || !m1_h || !v_h || !h_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  TOPT_CUDA(cudaMemcpyAsync(c->m0b, m0_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(c->m1b, m1_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(c->vb, v_h, c->vecN * 4, cudaMemcpyHostToDevice, st));
  topt_status r = eval_gradient(c, c->m0b, c->m1b, c->vb, nullptr, c->gcur, c->scur, pub(c, 4), intl(c, 4), st);
  if (r != TOPT_OK) return r;
  if (g_h) TOPT_CUDA(cudaMemcpyAsync(g_h, c->gcur, c->vecN * 4, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaMemcpyAsync(h_scalars, pub(c, 4), TOPT_NSCALARS * 8, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

topt_status topt_objective(topt_ctx* c, const float* m0, const float* m1, const float* v, double* d_scalars,
                           void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  forward_half(c, m0, m1, v, false, d_scalars, intl(c, 4), st);
  // reg = alpha/2 <v, L v>_h = h^d/2 sum v u,  u = alpha L v (fp64 chain)
  launch_vchain(c->g, v, c->Zv, c->utmp, c->p.alpha, c->p.reg_order, false, st);  // plain L, as in (1.1a)
  const float* bs[1] = {c->utmp};
  int np = 0;
  launch_multidot(v, bs, 1, c->vecN, c->partials, &np, st);
  launch_finalize_multi(c->partials, 0, 1, np, 0.5 * c->cellvol, d_scalars + TOPT_S_REG, st);
  launch_combine_obj(d_scalars, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_feet(topt_ctx* c, const float* v, float* delta_f, float* delta_a, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!v || (!delta_f && !delta_a)) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  launch_trace(c->g, v, delta_f, delta_a, nullptr, nullptr, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_forward(topt_ctx* c, const float* m0, const float* v, float* m_traj, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !v || !m_traj) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  forward_half(c, m0, m0, v, false, pub(c, 4), intl(c, 4), st);
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
  cudaStream_t st = (cudaStream_t)stream;
  const bool leray = c->p.model == TOPT_INCOMPRESSIBLE;
  launch_bchain(c->g, g, c->Z, c->p.alpha, c->p.reg_order, leray, st);
  int np = 0;
  launch_assemble(c->g, c->Z, leray, g, nullptr, nullptr, nullptr, nullptr, s, c->partials, &np, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_leray(topt_ctx* c, const float* u, float* out, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!u || !out) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  launch_bchain(c->g, u, c->Z, c->p.alpha, c->p.reg_order, true, st);
  int np = 0;
  launch_assemble(c->g, c->Z, true, nullptr, nullptr, nullptr, nullptr, out, nullptr, c->partials, &np, st);
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

topt_status topt_profile(topt_ctx* c, int32_t enable) {
  if (!c) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
  TOPT_CUDA(cudaDeviceSynchronize());
  for (auto& r : c->recs) { c->pool.push_back(r.a); c->pool.push_back(r.b); }
  c->recs.clear();
  for (int i = 0; i < 16; ++i) { c->pms[i] = 0.0; c->pbytes[i] = 0.0; c->plaunch[i] = 0; }
  c->prof = enable != 0;
  return TOPT_OK;
}

topt_status topt_kernel_stats(topt_ctx* c, int32_t cls, const char** name, double* ms, double* bytes,
                              int64_t* launches) {
  if (!c) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
  if (cls < 0 || cls >= K_NCLASS) return fail(TOPT_ERR_INVALID_ARG, "class out of range");
  for (auto& r : c->recs) {
    TOPT_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    TOPT_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    c->pms[r.cls] += t;
    c->pbytes[r.cls] += r.bytes;
    c->plaunch[r.cls] += r.launches;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  if (name) *name = kClassNames[cls];
  if (ms) *ms = c->pms[cls];
  if (bytes) *bytes = c->pbytes[cls];
  if (launches) *launches = c->plaunch[cls];
  return TOPT_OK;
}

int64_t topt_launch_count(void) { return (int64_t)launch_count(); }

topt_status topt_set_step_replay(topt_ctx* c, const double* rho, int32_t count) {
  if (!c || count < 0 || (count && !rho)) return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  c->replay.assign(rho, rho + count);
  return TOPT_OK;
}

// GA-NGMRES(w; sigma, tau) (Alg. 3) / GA-AA, host-driven.  u = alpha L v is carried with
// every iterate (q: u_q = u - rho P_0 g since alpha L s = -P_0 g; mixing is linear), so the
// evaluations inside the solve never apply L to a stored fp32 field.
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
  const bool leray = P.model == TOPT_INCOMPRESSIBLE;
  const double nF = (double)c->F;
  std::memset(rep, 0, sizeof(*rep));
  const double t0 = now();
  double t_pde = 0.0, t_ls = 0.0;
  int grad_evals = 0, obj_evals = 0, nsteps = 0;
  std::deque<double> replay(c->replay.begin(), c->replay.end());
  topt_status r;

  // history slot i: A = v (AA: r), B = g (AA: q), U = u (AA: u(q))
  auto slotA = [&](int i) { return c->hist + (size_t)(3 * i) * V; };
  auto slotB = [&](int i) { return c->hist + (size_t)(3 * i + 1) * V; };
  auto slotU = [&](int i) { return c->hist + (size_t)(3 * i + 2) * V; };
  std::deque<int> win;  // ring slots, most recent last
  std::vector<std::vector<double>> H(W1, std::vector<double>(W1, 0.0));  // <B_i, B_j> by slot
  auto take_slot = [&]() {
    int slot;
    if ((int)win.size() < W1) {
      slot = (int)win.size();
    } else {
      slot = win.front();
      win.pop_front();
    }
    return slot;
  };
  // push (a, b, u) and refresh the Gram row of b against the window
  auto push = [&](const float* a, const float* b, const float* u, bool gram) -> topt_status {
    const int slot = take_slot();
    TOPT_CUDA(cudaMemcpyAsync(slotA(slot), a, V * 4, cudaMemcpyDeviceToDevice, st));
    TOPT_CUDA(cudaMemcpyAsync(slotB(slot), b, V * 4, cudaMemcpyDeviceToDevice, st));
    TOPT_CUDA(cudaMemcpyAsync(slotU(slot), u, V * 4, cudaMemcpyDeviceToDevice, st));
    win.push_back(slot);
    if (!gram) return TOPT_OK;
    std::vector<const float*> bs;
    for (int s2 : win) bs.push_back(slotB(s2));
    std::vector<double> dd;
    topt_status rr = host_dots(c, slotB(slot), bs, dd, st);
    if (rr != TOPT_OK) return rr;
    for (size_t i = 0; i < win.size(); ++i) H[slot][win[i]] = H[win[i]][slot] = dd[i];
    return TOPT_OK;
  };

  // v^0, u^0 = alpha L v^0 (fp64 chain, once), g(v^0)
  TOPT_CUDA(cudaMemcpyAsync(c->vcur, v_inout, V * 4, cudaMemcpyDeviceToDevice, st));
  if (leray) leray_inplace(c, c->vcur, st);
  launch_vchain(c->g, c->vcur, c->Zv, c->ucur, P.alpha, P.reg_order, leray, st);
  double te = now();
  if ((r = eval_gradient(c, m0, m1, c->vcur, c->ucur, c->gcur, c->scur, pub(c, 0), intl(c, 0), st)) != TOPT_OK)
    return r;
  ++grad_evals;
  HostScalars cur, qs, ns;
  if ((r = fetch(c, 0, cur, st)) != TOPT_OK) return r;
  t_pde += now() - te;
  const double g0 = cur.pub(TOPT_S_GRAD_INF);
  rep->grad_inf0 = g0;
  if (!aa && (r = push(c->vcur, c->gcur, c->ucur, true)) != TOPT_OK) return r;

  // q-state helpers: v_q = v + rho s, u_q = u - rho (g - gbar)
  auto make_q = [&](double rho_) {
    launch_axpy(c->vcur, (float)rho_, c->scur, V, c->q, st);
    float cst[3] = {0.f, 0.f, 0.f};
    for (int a = 0; a < c->d; ++a) cst[a] = (float)(rho_ * cur.in(I_SUMG + a) / nF);
    launch_axpy_c(c->ucur, (float)(-rho_), c->gcur, V, c->d, cst, c->uq, st);
  };
  auto eval_q = [&]() -> topt_status {
    topt_status rr = eval_gradient(c, m0, m1, c->q, c->uq, c->gq, c->sq, pub(c, 2), intl(c, 2), st);
    if (rr != TOPT_OK) return rr;
    ++grad_evals;
    return fetch(c, 2, qs, st);
  };
  auto accept_q = [&]() {
    std::swap(c->vcur, c->q);
    std::swap(c->ucur, c->uq);
    std::swap(c->gcur, c->gq);
    std::swap(c->scur, c->sq);
    cur = qs;
  };
  auto eval_new = [&]() -> topt_status {
    if (leray) {
      leray_inplace(c, c->vnew, st);
      leray_inplace(c, c->unew, st);
    }
    topt_status rr = eval_gradient(c, m0, m1, c->vnew, c->unew, c->gnew, c->snew, pub(c, 3), intl(c, 3), st);
    if (rr != TOPT_OK) return rr;
    ++grad_evals;
    rr = fetch(c, 3, ns, st);
    if (rr != TOPT_OK) return rr;
    std::swap(c->vcur, c->vnew);
    std::swap(c->ucur, c->unew);
    std::swap(c->gcur, c->gnew);
    std::swap(c->scur, c->snew);
    cur = ns;
    return TOPT_OK;
  };

  double rho = 1.0;
  int k = 0;
  int exit_code = TOPT_ITER_CAP;
  while (P.max_iter > 0) {
    // ---- q(v^k): Armijo backtracking with memory (R12) ---------------------
    const double obj0 = cur.pub(TOPT_S_OBJ), gs = cur.pub(TOPT_S_GS);
    bool accepted = false;
    double rho_t = rho;
    te = now();
    if (!replay.empty()) {
      rho_t = replay.front();
      replay.pop_front();
      rho = rho_t;
      make_q(rho_t);
      accepted = true;
    } else {
      for (int t = 0; t <= P.max_backtracks; ++t) {
        make_q(rho_t);
        if ((r = trial_dist(c, m0, m1, c->q, pub(c, 1), intl(c, 1), st)) != TOPT_OK) return r;
        ++obj_evals;
        HostScalars ts;
        if ((r = fetch(c, 1, ts, st)) != TOPT_OK) return r;
        // reg(v + rho s) = reg + rho alpha<s, L v> + rho^2/2 alpha<s, L s>  (exact: quadratic)
        const double reg_t = cur.pub(TOPT_S_REG) + rho_t * cur.pub(TOPT_S_SLV) +
                             0.5 * rho_t * rho_t * cur.pub(TOPT_S_SLS);
        const double obj_t = ts.pub(TOPT_S_DIST) + reg_t;
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
    t_pde += now() - te;

    const int period = P.sigma + P.tau;
    const bool fp_step = P.ordering == TOPT_ORDER_GA ? (k % period >= P.sigma) : (k % period < P.tau);
    const int wk = std::min(k, P.window);
    if (!aa) {
      te = now();
      if ((r = eval_q()) != TOPT_OK) return r;  // g(q): both branches need it (R17)
      t_pde += now() - te;
      if (fp_step) {
        accept_q();
      } else {
        // LSQ (Alg. 3 line 8): columns C_i = g_q - g(v^{k-i}), i = 0..w_k (R13), from the
        // fp64 Gram: G_ij = <g_q,g_q> - <g_q,g_i> - <g_q,g_j> + <g_i,g_j>, rhs_i = <C_i, g_q>
        const double tl = now();
        const int m = (int)win.size();  // == w_k + 1
        std::vector<const float*> bs;
        for (int i = 0; i < m; ++i) bs.push_back(slotB(win[m - 1 - i]));  // i = 0 -> v^k
        bs.push_back(c->gq);
        std::vector<double> rd;
        if ((r = host_dots(c, c->gq, bs, rd, st)) != TOPT_OK) return r;
        const double gam = rd[m];
        std::vector<double> G(m * m), rhs(m);
        for (int i = 0; i < m; ++i) {
          const int si = win[m - 1 - i];
          rhs[i] = gam - rd[i];
          for (int j = 0; j < m; ++j) G[i * m + j] = gam - rd[i] - rd[j] + H[si][win[m - 1 - j]];
        }
        std::vector<double> beta = lsq_from_gram(m, G, rhs);
        t_ls += now() - tl;
        // v^{k+1} = q + sum beta_i (q - v^{k-i})  (Alg. 3 line 9), same combination for u
        std::vector<const float*> vs, us;
        for (int i = 0; i < m; ++i) {
          vs.push_back(slotA(win[m - 1 - i]));
          us.push_back(slotU(win[m - 1 - i]));
        }
        launch_mix(c->q, vs.data(), beta.data(), m, V, c->vnew, st);
        launch_mix(c->uq, us.data(), beta.data(), m, V, c->unew, st);
        te = now();
        if ((r = eval_new()) != TOPT_OK) return r;
        t_pde += now() - te;
        ++nsteps;
      }
      (void)wk;
      if ((r = push(c->vcur, c->gcur, c->ucur, true)) != TOPT_OK) return r;
    } else {
      // AA (Alg. 2): r_k = v^k - q(v^k); LSQ over r_k - r_{k-i}, i = 1..w_k; mix q-images
      launch_sub(c->vcur, c->q, V, c->vt, st);  // r_k
      const int m = std::min((int)win.size(), wk);
      if (!fp_step && m > 0) {
        const double tl = now();
        std::vector<const float*> bs;
        for (int i = 0; i < m; ++i) bs.push_back(slotA(win[win.size() - 1 - i]));
        bs.push_back(c->vt);
        std::vector<double> rd;
        if ((r = host_dots(c, c->vt, bs, rd, st)) != TOPT_OK) return r;
        const double gam = rd[m];
        std::vector<double> G(m * m), rhs(m);
        for (int i = 0; i < m; ++i) {
          std::vector<const float*> b2;
          for (int j = 0; j < m; ++j) b2.push_back(slotA(win[win.size() - 1 - j]));
          std::vector<double> row;
          if ((r = host_dots(c, slotA(win[win.size() - 1 - i]), b2, row, st)) != TOPT_OK) return r;
          rhs[i] = gam - rd[i];
          for (int j = 0; j < m; ++j) G[i * m + j] = gam - rd[i] - rd[j] + row[j];
        }
        std::vector<double> xi = lsq_from_gram(m, G, rhs);
        t_ls += now() - tl;
        std::vector<const float*> qv, qu;
        for (int i = 0; i < m; ++i) {
          qv.push_back(slotB(win[win.size() - 1 - i]));
          qu.push_back(slotU(win[win.size() - 1 - i]));
        }
        launch_mix(c->q, qv.data(), xi.data(), m, V, c->vnew, st);
        launch_mix(c->uq, qu.data(), xi.data(), m, V, c->unew, st);
        if ((r = push(c->vt, c->q, c->uq, false)) != TOPT_OK) return r;
        te = now();
        if ((r = eval_new()) != TOPT_OK) return r;
        t_pde += now() - te;
        ++nsteps;
      } else {
        if ((r = push(c->vt, c->q, c->uq, false)) != TOPT_OK) return r;
        te = now();
        if ((r = eval_q()) != TOPT_OK) return r;
        t_pde += now() - te;
        accept_q();
      }
    }
    ++k;
    const double gi = cur.pub(TOPT_S_GRAD_INF);
    if (!std::isfinite(gi) || !std::isfinite(cur.pub(TOPT_S_OBJ)))
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
  rep->obj = cur.pub(TOPT_S_OBJ);
  rep->dist = cur.pub(TOPT_S_DIST);
  rep->reg = cur.pub(TOPT_S_REG);
  rep->grad_inf = cur.pub(TOPT_S_GRAD_INF);
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
