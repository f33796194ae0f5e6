// api.cu — C ABI of libtopt: context, workspace, gradient evaluation and the GA-NGMRES
// driver (host logic; every field operation runs in the kernels of kernels_*.cu, every
// exchange between z-slabs in dist.cu).
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
#include <functional>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace topt;

namespace topt {
bool comm_halo(topt_ctx* c, const std::vector<float*>& base, int nf, size_t fstride, cudaStream_t st);
bool comm_z2y(topt_ctx* c, const std::vector<const char*>& src, const std::vector<char*>& dst, size_t eb,
              cudaStream_t st);
bool comm_y2z(topt_ctx* c, const std::vector<const char*>& src, const std::vector<char*>& dst, size_t eb,
              cudaStream_t st);
bool comm_allreduce(topt_ctx* c, const std::vector<double*>& ptr, int count, bool is_max, cudaStream_t st);
bool comm_p2p_ready(const topt_ctx* c);
char* comm_peer(const topt_ctx* c, const void* p, int q);
bool comm_fence(topt_ctx* c, cudaStream_t st);
int comm_agree_min(topt_ctx* c, int v);
bool comm_window(topt_ctx* c, const std::vector<const float*>& src, size_t fs, int nf, int zw, cudaStream_t st);
}  // namespace topt

namespace {
// Destroy every captured evaluation graph (workspace, transport or peer mappings changed).
void drop_graphs(topt_ctx* c) {
  for (auto& ge : c->graphs) cudaGraphExecDestroy(ge.exec);
  c->graphs.clear();
}

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
  if (world < 1 || world > 64 || !pow2(world))
    return fail(TOPT_ERR_INVALID_ARG, "world must be a power of two <= 64");
  if (world > 1) {
    if (p->dim != 3) return fail(TOPT_ERR_INVALID_ARG, "dim == 2 runs on one rank");
    if (p->n[2] % world || p->n[1] % world) return fail(TOPT_ERR_INVALID_ARG, "n[1] and n[2] must divide by world");
    if (p->n[2] / world < kSlabHalo) return fail(TOPT_ERR_INVALID_ARG, "n[2] / world must be >= 4 (halo)");
    if (p->n[0] < 32 || p->n[1] % 8) return fail(TOPT_ERR_UNSUPPORTED, "z-slabs need n[0] >= 32 and n[1] % 8 == 0");
  }
  return TOPT_OK;
}

topt_status topt_create(const topt_params* p, int32_t rank, int32_t world, const uint8_t* id, int32_t device,
                        topt_ctx** out) {
  if (!out) return fail(TOPT_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  topt_status s = validate(p, world);
  if (s != TOPT_OK) return s;
  if (rank < 0 || rank >= world) return fail(TOPT_ERR_INVALID_ARG, "rank out of range");
  const bool emulate = world > 1 && id == nullptr;
  if (emulate && rank != 0) return fail(TOPT_ERR_INVALID_ARG, "emulated z-slabs (id == NULL) run as rank 0");
#ifndef TOPT_WITH_NCCL
  if (world > 1 && !emulate) return fail(TOPT_ERR_UNSUPPORTED, "libtopt built without NCCL");
#endif
  TOPT_CUDA(cudaSetDevice(device));
  auto* c = new topt_ctx();
  c->p = *p;
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->d = p->dim;
  c->nzg = p->dim == 3 ? p->n[2] : 1;
  c->comm.P = world;
  c->comm.nloc = emulate ? world : 1;
#ifdef TOPT_WITH_NCCL
  if (world > 1 && !emulate) {
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    if (ncclCommInitRank(&c->comm.nccl, world, u, rank) != ncclSuccess) {
      delete c;
      return fail(TOPT_ERR_NCCL, "ncclCommInitRank failed");
    }
  }
#endif
  c->dt = 1.0 / p->nt;
  c->cellvol = 1.0;
  for (int a = 0; a < c->d; ++a) {
    c->h[a] = 2.0 * M_PI / p->n[a];
    c->cellvol *= c->h[a];
  }
  c->wts.assign(p->nt + 1, c->dt);
  c->wts.front() = c->wts.back() = 0.5 * c->dt;
  const int nzl = c->nzg / world;
  c->slabs.resize(c->comm.nloc);
  for (int si = 0; si < c->comm.nloc; ++si) {
    Slab& sl = c->slabs[si];
    sl.index = emulate ? si : rank;
    Geom& g = sl.g;
    g.d = p->dim;
    g.nx = p->n[0];
    g.ny = p->n[1];
    g.nz = nzl;
    g.lx = ilog2(g.nx);
    g.ly = ilog2(g.ny);
    g.lz = ilog2(g.nz);
    g.F = (size_t)g.nx * g.ny * g.nz;
    g.cx = (float)(c->dt / c->h[0]);
    g.cy = (float)(c->dt / c->h[1]);
    g.cz = c->d == 3 ? (float)(c->dt / c->h[2]) : 0.f;
    g.zh = world > 1 ? kSlabHalo : 0;
    g.ky0 = 0;
    g.nyg = 0;
    g.haloerr = nullptr;
    sl.gy = g;  // y-slab layout of the z passes: [nz][ny/P][nx]
    sl.gy.ny = g.ny / world;
    sl.gy.ly = ilog2(sl.gy.ny);
    sl.gy.nz = c->nzg;
    sl.gy.lz = ilog2(c->nzg);
    sl.gy.zh = 0;
    sl.gy.ky0 = sl.index * sl.gy.ny;
    sl.gy.nyg = g.ny;
    sl.F = g.F;
    sl.plane = (size_t)g.nx * g.ny;
    sl.Fh = g.F + 2 * (size_t)g.zh * sl.plane;
  }
  c->F = c->slabs[0].F;
  c->vecN = (size_t)c->d * c->F;
  // window capacity: (nzl + 2 hcap) >= nz + 3 planes cover every periodic foot position
  c->hcap = world > 1 ? (c->nzg - nzl + 4) / 2 : 0;
  // workspace size per slab
  const Slab& s0 = c->slabs[0];
  const size_t F = s0.F, Fh = s0.Fh, V = c->vecN, S1 = p->nt + 1, W1 = p->window + 1;
  size_t b = 0;
  auto add = [&](size_t bytes) { b += align256(bytes); };
  add(S1 * Fh * 4); add(S1 * Fh * 4);                          // m_traj, lam_traj
  add(world > 1 ? c->d * Fh * 4 : 0); add(Fh * 4);             // vh, divv
  add(V * 4); add(V * 4); add(F * 4); add(V * 4); add(V * 4);  // df, da, E, b, utmp
  add(4 * F * 8); add(3 * F * 16);                             // Z, Zv
  if (world > 1) {
    add(4 * F * 8); add(3 * F * 16);                           // Zy, Zvy
    add(2 * S1 * F * 4); add(2 * F * 4);                       // ytraj, ytmp
    add(16 * F);                                               // sendbuf
    add(3 * (F + 2 * (size_t)c->hcap * s0.plane) * 4);         // wide-halo window
  }
  add(F * 4); add(F * 4); add(V * 4); add(V * 4);              // m0b, m1b, vb, vt
  for (int i = 0; i < 12; ++i) add(V * 4);                     // solver vectors
  add(3 * W1 * V * 4);                                         // history
  add((size_t)kNumSlots * kMaxPartials * 8);
  add(5 * kSet * 8);
  add(kMaxVecs * kMaxVecs * 8);
  add(256);                                                    // halo error flag
  c->slab_bytes = b;
  c->ws_need = b * c->comm.nloc;
  upload_twiddles();
  if (c->comm.P == 1) {  // side stream for v-only work (eval_gradient), see eval_gradient
#ifndef TOPT_SIDE_PRIO
#define TOPT_SIDE_PRIO 0  // 1: high-priority side stream (measured: no change, 151.6 vs 151.8 evals/s)
#endif
    // high priority: the block scheduler hands SMs freed by the SL grids to the side stream's blocks
    // first, so div v and the fp64 v transforms interleave with the sweeps instead of trailing them
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, TOPT_SIDE_PRIO ? hi : lo);
    cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_div, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_u, cudaEventDisableTiming);
  }
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
  for (auto& ge : ctx->graphs) cudaGraphExecDestroy(ge.exec);
  if (ctx->gcap) {
    cudaStreamSynchronize(ctx->gcap);
    cudaStreamDestroy(ctx->gcap);
    cudaEventDestroy(ctx->ev_gcap);
  }
  if (ctx->h_in) {
    for (cudaStream_t x : {ctx->h_in, ctx->h_comp, ctx->h_out}) {
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
    cudaEventDestroy(ctx->ev_hfork);
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {ctx->ev_hin[i], ctx->ev_hfree[i], ctx->ev_hdone[i], ctx->ev_hout[i]}) cudaEventDestroy(e);
  }
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_div);
    cudaEventDestroy(ctx->ev_u);
  }
#ifdef TOPT_WITH_NCCL
  if (ctx->comm.nccl) ncclCommDestroy(ctx->comm.nccl);
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
  // peer mappings refer to the previous workspaces: transport 1 needs topt_set_peer_workspaces again
  c->comm.peer_ws.clear();
  c->comm.transport = 0;
  drop_graphs(c);  // they bake the old workspace in
  const int world = c->world;
  for (int si = 0; si < c->comm.nloc; ++si) {
    Slab& sl = c->slabs[si];
    const size_t F = sl.F, Fh = sl.Fh, V = c->vecN, S1 = c->p.nt + 1, W1 = c->p.window + 1;
    char* q = c->ws + si * c->slab_bytes;
    auto take = [&](size_t bytes_) { char* r = q; q += align256(bytes_); return r; };
    sl.m_traj = (float*)take(S1 * Fh * 4);
    sl.lam_traj = (float*)take(S1 * Fh * 4);
    sl.vh = (float*)take(world > 1 ? c->d * Fh * 4 : 0);
    sl.divv = (float*)take(Fh * 4);
    sl.df = (float*)take(V * 4);
    sl.da = (float*)take(V * 4);
    sl.E = (float*)take(F * 4);
    sl.b = (float*)take(V * 4);
    sl.utmp = (float*)take(V * 4);
    sl.Z = (float2*)take(4 * F * 8);
    sl.Zv = (double2*)take(3 * F * 16);
    if (world > 1) {
      sl.Zy = (float2*)take(4 * F * 8);
      sl.Zvy = (double2*)take(3 * F * 16);
      sl.ytraj = (float*)take(2 * S1 * F * 4);
      sl.ytmp = (float*)take(2 * F * 4);
      sl.sendbuf = take(16 * F);
      sl.win = (float*)take(3 * (F + 2 * (size_t)c->hcap * sl.plane) * 4);
    }
    sl.m0b = (float*)take(F * 4);
    sl.m1b = (float*)take(F * 4);
    sl.vb = (float*)take(V * 4);
    sl.vt = (float*)take(V * 4);
    float** vecs[12] = {&sl.vcur, &sl.gcur, &sl.scur, &sl.q,    &sl.gq,   &sl.sq,
                        &sl.vnew, &sl.gnew, &sl.snew, &sl.ucur, &sl.uq,   &sl.unew};
    for (auto pp : vecs) *pp = (float*)take(V * 4);
    sl.hist = (float*)take(3 * W1 * V * 4);
    sl.partials = (double*)take((size_t)kNumSlots * kMaxPartials * 8);
    sl.sc = (double*)take(5 * kSet * 8);
    sl.dots = (double*)take(kMaxVecs * kMaxVecs * 8);
    sl.haloerr = (int*)take(256);
    sl.amax = (unsigned*)(sl.haloerr + 1);
    sl.amaxd = (double*)sl.haloerr + 1;
    sl.g.haloerr = sl.haloerr;
    sl.gy.haloerr = sl.haloerr;
  }
  for (auto& sl : c->slabs) TOPT_CUDA(cudaMemset(sl.haloerr, 0, sizeof(int)));
  return TOPT_OK;
}

topt_status topt_set_transport(topt_ctx* ctx, int32_t transport) {
  if (!ctx) return fail(TOPT_ERR_INVALID_ARG, "NULL context");
  if (transport != 0 && transport != 1) return fail(TOPT_ERR_INVALID_ARG, "transport must be 0 or 1");
  const Comm& cm = ctx->comm;
  if (cm.P > 1 && !cm.emulated()) {
    // collective: the ranks' choices decide which collectives each issues, so they must agree —
    // transport 1 only if EVERY rank asked for it and holds the peer mappings
    if (!ctx->ws) return fail(TOPT_ERR_WORKSPACE, "bind the workspace before topt_set_transport");
    const int mine = transport == 1 && (int)cm.peer_ws.size() == cm.P ? 1 : 0;
    transport = comm_agree_min(ctx, mine);
  }
  if (ctx->comm.transport != transport) drop_graphs(ctx);  // captured z-slab segments bake the transport in
  ctx->comm.transport = transport;
  return TOPT_OK;
}

int32_t topt_get_transport(const topt_ctx* ctx) { return ctx ? ctx->comm.transport : -1; }

topt_status topt_set_peer_workspaces(topt_ctx* ctx, void* const* bases, int32_t count) {
  if (!ctx) return fail(TOPT_ERR_INVALID_ARG, "NULL context");
  if (count == 0) {
    ctx->comm.peer_ws.clear();
    drop_graphs(ctx);
    return TOPT_OK;
  }
  if (count != ctx->comm.P || !bases) return fail(TOPT_ERR_INVALID_ARG, "count must equal the world size");
  drop_graphs(ctx);  // captured P2P segments bake the peer addresses in
  ctx->comm.peer_ws.assign(count, nullptr);
  for (int r = 0; r < count; ++r) ctx->comm.peer_ws[r] = static_cast<char*>(bases[r]);
  return TOPT_OK;
}

topt_status topt_local_slab(const topt_ctx* ctx, int32_t* z0, int32_t* nz) {
  if (!ctx || !z0 || !nz) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  const bool emu = ctx->comm.P > 1 && ctx->comm.emulated();
  *z0 = emu ? 0 : ctx->slabs[0].index * ctx->slabs[0].g.nz;
  *nz = ctx->d == 3 ? (emu ? ctx->nzg : ctx->slabs[0].g.nz) : 1;
  return TOPT_OK;
}

}  // extern "C"

// ======================================================================================
// Internal orchestration (loops over the local slabs; exchanges through dist.cu)
// ======================================================================================
namespace {

// Kernel classes for topt_kernel_stats; bytes are ALGORITHMIC (each operand read once,
// each result written once per launch group).  K_SL_STEP: every interior SL
// step of both sweeps (one kernel); the last forward step (fused mismatch) is its own class.
enum KClass { K_TRACE, K_SL_STEP, K_SL_LAST, K_EFACTOR, K_DIV, K_BODY, K_VCHAIN, K_BCHAIN, K_ASSEMBLE, K_COMM,
              K_MISC, K_GRAM, K_MIX, K_NCLASS };
const char* kClassNames[K_NCLASS] = {"sl_trace",   "sl_step",        "sl_step_last", "efactor",  "div_v",
                                     "body_force", "vchain_alphaLv", "bchain_fft",   "assemble", "comm",
                                     "misc",       "ngmres_gram",    "ngmres_mix"};

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
int P_of(const topt_ctx* c) { return c->comm.P; }
double ntot(const topt_ctx* c) { return (double)c->F * c->comm.P; }
float* local(const Slab& s, float* base) { return base + (size_t)s.g.zh * s.plane; }

// Per-slab inputs / outputs of one evaluation.
struct Io {
  const float* m0;
  const float* m1;
  const float* v;   // d*F local layout
  const float* u;   // alpha L v (d*F) or null
  float* g;
  float* s;
  double* scal;     // public scalars
  double* isc;      // internal scalars
};

std::vector<double*> pubs(std::vector<Io>& io, int off) {
  std::vector<double*> r;
  for (auto& x : io) r.push_back(x.scal + off);
  return r;
}
std::vector<double*> intls(std::vector<Io>& io, int off) {
  std::vector<double*> r;
  for (auto& x : io) r.push_back(x.isc + off);
  return r;
}

// z-slab <-> y-slab transposes of one field per slab
template <typename T>
bool tz2y(topt_ctx* c, const std::vector<T*>& src, const std::vector<T*>& dst, cudaStream_t st) {
  std::vector<const char*> s;
  std::vector<char*> d;
  for (auto p : src) s.push_back((const char*)p);
  for (auto p : dst) d.push_back((char*)p);
  Prof pr(c, K_COMM, 2.0 * sizeof(T) * c->F * c->comm.nloc, 0, st);
  return comm_z2y(c, s, d, sizeof(T), st);
}
template <typename T>
bool ty2z(topt_ctx* c, const std::vector<T*>& src, const std::vector<T*>& dst, cudaStream_t st) {
  std::vector<const char*> s;
  std::vector<char*> d;
  for (auto p : src) s.push_back((const char*)p);
  for (auto p : dst) d.push_back((char*)p);
  Prof pr(c, K_COMM, 2.0 * sizeof(T) * c->F * c->comm.nloc, 0, st);
  return comm_y2z(c, s, d, sizeof(T), st);
}
bool halo(topt_ctx* c, std::function<float*(Slab&)> base, int nf, size_t fstride, cudaStream_t st) {
  if (P_of(c) == 1) return true;
  std::vector<float*> b;
  for (auto& sl : c->slabs) b.push_back(base(sl));
  const Slab& s0 = c->slabs[0];
  Prof pr(c, K_COMM, 4.0 * nf * s0.g.zh * s0.plane * 4.0 * c->comm.nloc, 0, st);
  return comm_halo(c, b, nf, fstride, st);
}

// ---- z-slab window sizing ("halo exchange sized from max|v|*dt"; P:136 no CFL cap)
// Device part: max |x| over every slab's F floats of a(slab) and b(slab) (b may be null),
// all-reduced (max) into slab 0's amaxd.
void zmax_dev(topt_ctx* c, std::function<const float*(Slab&)> a, std::function<const float*(Slab&)> b,
              cudaStream_t st) {
  std::vector<double*> slots;
  for (auto& sl : c->slabs) {
    cudaMemsetAsync(sl.amax, 0, sizeof(unsigned), st);
    launch_absmax(a(sl), b ? b(sl) : nullptr, sl.F, sl.amax, st);
    launch_uint_as_float_to_double(sl.amax, sl.amaxd, st);
    slots.push_back(sl.amaxd);
  }
  comm_allreduce(c, slots, 1, true, st);
}
// Host part: read it (synchronises `st`; z-slabs only, a few microseconds per evaluation).
double zmax_read(topt_ctx* c, cudaStream_t st) {
  double h = 0.0;
  cudaMemcpyAsync(&h, c->slabs[0].amaxd, sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}
// Half-width of the input window for feet of at most D cells in z: the tricubic stencil of a
// foot z + delta spans planes floor(z + delta) - 1 .. + 2, so |delta| <= D needs floor(D) + 2
// planes per side.  0 = the stored kSlabHalo planes suffice (D < 3); beyond the capacity the
// window covers a whole period and feet are wrapped into it (nzw).
void size_window(const topt_ctx* c, double D, int& zw, bool& wrap) {
  const double need = std::isfinite(D) ? std::floor(D * (1.0 + 1e-6)) + 2.0 : 1e30;
  if (need <= kSlabHalo) {
    zw = 0;
    wrap = false;
    return;
  }
  zw = (int)std::min<double>(need, c->hcap);
  wrap = need > c->hcap;
}
Geom in_geom(const topt_ctx* c, const Slab& sl, int zw, bool wrap) {
  if (!zw) return sl.g;
  Geom g = sl.g;
  g.zh = zw;
  g.nzw = wrap ? c->nzg : 0;
  return g;
}

// The two window decisions of a z-slab evaluation as one integer (zw, wrap): point 0 sizes the
// trace input from max |v_z| (the midpoint displacement dt/2 v_z/h_z is exact at the nodes),
// point 1 the SL-step inputs from max |delta_z| over the feet.
int window_code(int zw, bool wrap) { return 2 * zw + (wrap ? 1 : 0); }
void window_of(int code, int& zw, bool& wrap) {
  zw = code >> 1;
  wrap = (code & 1) != 0;
}
int decision_of(const topt_ctx* c, double h, int point) {
  const double D = point == 0 ? 0.5 * h * (double)c->slabs[0].g.cz : h;
  int zw = 0;
  bool wrap = false;
  size_window(c, D, zw, wrap);
  return window_code(zw, wrap);
}

// ---- segmented CUDA-graph capture of z-slab evaluations (P > 1) --------------------------
const int kMaxGraphs = 32;
const int kSlabSegs = 3;  // [v halo, max|v_z|] | [trace, max|delta_z|] | [rest of the evaluation]
void seg_key(const void* key[8], const void* const base[6], int seg, const std::vector<int>& dec) {
  key[0] = (const void*)(uintptr_t)(0x5e60 + seg);
  for (int i = 0; i < 6; ++i) key[1 + i] = base[i];
  uintptr_t d = 0;
  for (size_t i = 0; i < dec.size() && (int)i < seg; ++i) d |= (uintptr_t)(dec[i] & 0xfffff) << (20 * i);
  key[7] = (const void*)d;
}
topt_ctx::GraphEntry* find_graph(topt_ctx* c, const void* const key[8]) {
  for (auto& ge : c->graphs)
    if (std::equal(ge.key, ge.key + 8, key)) return &ge;
  return nullptr;
}
void cache_graph(topt_ctx* c, const void* const key[8], cudaGraphExec_t exec, long long nlaunch) {
  if (topt_ctx::GraphEntry* old = find_graph(c, key)) {
    cudaGraphExecDestroy(old->exec);
    old->exec = exec;
    old->nlaunch = nlaunch;
    return;
  }
  if ((int)c->graphs.size() >= kMaxGraphs) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  topt_ctx::GraphEntry ge;
  std::copy(key, key + 8, ge.key);
  ge.exec = exec;
  ge.nlaunch = nlaunch;
  c->graphs.push_back(ge);
}
// End the segment being captured on gcap (index = decisions taken so far): instantiate and
// cache it, launch it on the user stream when `launch` (segments already replayed by this
// evaluation are only re-cached), and unless `last` begin capturing the next segment.
void seg_end(topt_ctx* c, bool launch, bool last) {
  topt_ctx::SegCap& s = c->segc;
  const int seg = (int)s.dec.size();
  const long long nl = launch_count() - s.l0;
  launch_count_add(-nl);  // captured, not launched
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  if (cudaStreamEndCapture(c->gcap, &graph) != cudaSuccess || !graph ||
      cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess)
    s.err = true;
  if (graph) cudaGraphDestroy(graph);
  if (!s.err) {
    const void* key[8];
    seg_key(key, s.base, seg, s.dec);
    cache_graph(c, key, exec, nl);
    if (launch) {
      if (cudaGraphLaunch(exec, s.user) != cudaSuccess) s.err = true;
      launch_count_add(nl);
    }
  }
  s.l0 = launch_count();
  if (!last && !s.err && cudaStreamBeginCapture(c->gcap, cudaStreamCaptureModeRelaxed) != cudaSuccess) s.err = true;
}
// One window decision (point 0 or 1) of a z-slab evaluation: the device part on `st`, then the
// host read.  Under segmented capture the segment ends here: it is launched on the user stream
// and the decision read there — or, for a segment this evaluation already replayed, the
// decision it took is reused.
int window_decision(topt_ctx* c, std::function<const float*(Slab&)> a, std::function<const float*(Slab&)> b,
                    int point, cudaStream_t st) {
  zmax_dev(c, a, b, st);
  topt_ctx::SegCap& s = c->segc;
  if (!s.on) return decision_of(c, zmax_read(c, st), point);
  const size_t i = s.dec.size();
  int d = 0;
  if (i < s.known.size()) {
    seg_end(c, false, false);
    d = s.known[i];
  } else {
    seg_end(c, true, false);
    d = s.err ? 0 : decision_of(c, zmax_read(c, s.user), point);
  }
  s.dec.push_back(d);
  return d;
}
// Input of an interpolation over nf fields (field f of slab s at base(s) + f * fstride, halo'd
// layout): the stored halo refreshed (zw == 0) or the window gathered into s.win from the LOCAL
// planes of every slab (multi-hop).  The kernel then reads in_ptr(...) with in_geom(...).
bool sl_input(topt_ctx* c, std::function<float*(Slab&)> base, int nf, size_t fstride, int zw, cudaStream_t st) {
  if (P_of(c) == 1) return true;
  if (zw == 0) return halo(c, base, nf, fstride, st);
  std::vector<const float*> src;
  for (auto& sl : c->slabs) src.push_back(local(sl, base(sl)));
  const Slab& s0 = c->slabs[0];
  Prof pr(c, K_COMM, 2.0 * nf * (s0.F + 2.0 * zw * s0.plane) * 4.0 * c->comm.nloc, 0, st);
  return comm_window(c, src, fstride, nf, zw, st);
}
const float* in_ptr(const Slab& sl, const float* base, int zw) { return zw ? sl.win : base; }

// div v = sum_a d_a v_a (R3), into the local planes of divv; halo refreshed
void compute_div(topt_ctx* c, std::vector<Io>& io, cudaStream_t st) {
  const int P = P_of(c);
  double one = 1.0;
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    const int na = P > 1 ? 2 : c->d;  // z handled by the transpose below when P > 1
    for (int a = 0; a < na; ++a) {
      DerivArgs da{io[si].v + a * sl.F, 0, nullptr, 0, &one, 1, a == 0 ? 0.f : 1.f, local(sl, sl.divv)};
      launch_deriv_accum(sl.g, a, da, st);
    }
  }
  if (P > 1) {
    std::vector<float*> src, dst, ysrc, back;
    for (size_t si = 0; si < c->slabs.size(); ++si) {  // v_z from the workspace copy (P2P-pullable)
      Slab& sl = c->slabs[si];
      src.push_back(local(sl, sl.vh + 2 * sl.Fh));
      dst.push_back(sl.ytmp);
    }
    tz2y(c, src, dst, st);
    for (auto& sl : c->slabs) {
      DerivArgs da{sl.ytmp, 0, nullptr, 0, &one, 1, 0.f, sl.ytmp + sl.F};
      launch_deriv_accum(sl.gy, 2, da, st);
      ysrc.push_back(sl.ytmp + sl.F);
      back.push_back(sl.utmp);
    }
    ty2z(c, ysrc, back, st);
    for (auto& sl : c->slabs) launch_axpy(local(sl, sl.divv), 1.0f, sl.utmp, sl.F, local(sl, sl.divv), st);
    halo(c, [](Slab& s) { return s.divv; }, 1, 0, st);
  }
}

// P2P transport, 3D non-Leray: the tables of nf fields (field f of slab q at base(slab) + f F)
// for the in-place last-axis passes on the distributed slabs; false when not applicable
template <typename T, typename Base>
static bool remote_fields(topt_ctx* c, Base base, int nf, std::vector<const void*>& tab) {
  const int P = P_of(c);
  if (P == 1 || c->d != 3 || c->p.model == TOPT_INCOMPRESSIBLE || !comm_p2p_ready(c)) return false;
  const bool emu = c->comm.emulated();
  tab.assign((size_t)nf * P, nullptr);
  for (int f = 0; f < nf; ++f)
    for (int q = 0; q < P; ++q) {
      Slab& sq = emu ? c->slabs[q] : c->slabs[0];
      tab[(size_t)f * P + q] = comm_peer(c, (const T*)base(sq) + (size_t)f * c->F, q);
    }
  return true;
}

// u = alpha L v by the fp64 v-chain (P_L first for incompressible, R9) into utmp; io[].u := utmp
void run_vchain(topt_ctx* c, std::vector<Io>& io, cudaStream_t st) {
  const int P = P_of(c);
  const size_t F = c->F;
  const double F4 = 4.0 * F, d = c->d;
  const bool leray = c->p.model == TOPT_INCOMPRESSIBLE;
  const double half = c->d == 3 ? 2.0 : 1.0;
  const double n_all = ntot(c);
  {
    const double nin = leray ? d : half, nout = half, F16 = 16.0 * F;
    const double bytes = d * F4 + nin * F16 + (c->d == 3 ? 2 * nin * F16 + 2 * nout * F16 : 0.0) +
                         (nin + nout) * F16 + nout * F16 + d * F4;
    Prof pr(c, K_VCHAIN, bytes * c->comm.nloc, c->d == 3 ? 5 : 3, st);
    const int vin = vchain_nin(c->slabs[0].g, leray), vout = vchain_nout(c->slabs[0].g);
    for (size_t si = 0; si < c->slabs.size(); ++si) {
      Slab& sl = c->slabs[si];
      double2* Z[3] = {sl.Zv, sl.Zv + F, sl.Zv + 2 * F};
      vchain_xy(sl.g, io[si].v, Z, leray, st);
    }
    std::vector<const void*> rtab;
    if (remote_fields<double2>(c, [](Slab& s) { return s.Zv; }, vin, rtab)) {
      comm_fence(c, st);  // every rank's x, y passes are complete
      for (auto& sl : c->slabs)
        vchain_last_remote(sl.gy, rtab.data(), P, sl.g.nz, sl.plane, c->p.alpha, c->p.reg_order, n_all, st);
      comm_fence(c, st);  // every rank's z lines are transformed
    } else {
      if (P > 1)
        for (int f = 0; f < vin; ++f) {
          std::vector<double2*> a, b;
          for (auto& sl : c->slabs) { a.push_back(sl.Zv + f * F); b.push_back(sl.Zvy + f * F); }
          tz2y(c, a, b, st);
        }
      for (auto& sl : c->slabs) {
        double2* base = P > 1 ? sl.Zvy : sl.Zv;
        double2* Z[3] = {base, base + F, base + 2 * F};
        vchain_last(P > 1 ? sl.gy : sl.g, Z, c->p.alpha, c->p.reg_order, leray, n_all, st);
      }
      if (P > 1)
        for (int f = 0; f < vout; ++f) {
          std::vector<double2*> a, b;
          for (auto& sl : c->slabs) { a.push_back(sl.Zvy + f * F); b.push_back(sl.Zv + f * F); }
          ty2z(c, a, b, st);
        }
    }
    for (size_t si = 0; si < c->slabs.size(); ++si) {
      Slab& sl = c->slabs[si];
      double2* Z[3] = {sl.Zv, sl.Zv + F, sl.Zv + 2 * F};
      vchain_inv(sl.g, Z, sl.utmp, st);
      io[si].u = sl.utmp;
    }
  }
}

// Merged v/b chain (kernels_spectral.cu gchain_*): one slab, non-Leray, u not supplied and
// not wanted by the caller.  Only the forward transform of v runs in fp64; g^ = alpha L v^ +
// b^ and p^ are formed at the last-axis pass and share the fp32 inverse passes.
bool merged_chain(const topt_ctx* c, const std::vector<Io>& io) {
  return c->comm.P == 1 && c->p.model != TOPT_INCOMPRESSIBLE && io[0].u == nullptr && !c->want_u;
}
// fp64 forward x (and y) passes of v into Zv
void vchain_fwd(topt_ctx* c, std::vector<Io>& io, cudaStream_t st) {
  const double F = (double)c->F, d = c->d, half = c->d == 3 ? 2.0 : 1.0;
  Prof pr(c, K_VCHAIN, d * 4.0 * F + half * 16.0 * F + (c->d == 3 ? 2.0 * half * 16.0 * F : 0.0), c->d == 3 ? 2 : 1,
          st);
  Slab& sl = c->slabs[0];
  double2* Z[3] = {sl.Zv, sl.Zv + sl.F, sl.Zv + 2 * sl.F};
  vchain_xy(sl.g, io[0].v, Z, false, st);
}

// Forward half: feet (R6), static factor (continuity, R7), m^0..m^S, lam^S = m1 - m^S
// (R1/R8), dist -> scal[DIST], sum_x v_c -> isc[I_SUMV..] (all-reduced).
void forward_half(topt_ctx* c, std::vector<Io>& io, bool want_adj, cudaStream_t st) {
  const int S = c->p.nt, P = P_of(c);
  const double F4 = 4.0 * c->F, d = c->d;
  if (P > 1) {  // halo'd copy of v for the trace
    for (size_t si = 0; si < c->slabs.size(); ++si) {
      Slab& sl = c->slabs[si];
      for (int a = 0; a < c->d; ++a)
        cudaMemcpyAsync(local(sl, sl.vh + a * sl.Fh), io[si].v + a * sl.F, sl.F * 4, cudaMemcpyDeviceToDevice, st);
    }
    // trace input: midpoint displacements dt/2 v_z/h_z at the nodes (exact, no interpolation)
    window_of(window_decision(c, [](Slab& s) { return (const float*)local(s, s.vh + 2 * s.Fh); }, nullptr, 0, st),
              c->zw_v, c->wrap_v);
    sl_input(c, [](Slab& s) { return s.vh; }, c->d, c->slabs[0].Fh, c->zw_v, st);
  }
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    int np = 0;
    {
      Prof pr(c, K_TRACE, (d + d * (want_adj ? 2 : 1)) * F4, 1, st);
      launch_trace(in_geom(c, sl, c->zw_v, c->wrap_v), P > 1 ? in_ptr(sl, sl.vh, c->zw_v) : io[si].v, sl.df,
                   want_adj ? sl.da : nullptr, sl.partials, &np, st);
    }
    Prof pr(c, K_MISC, 0.0, 1, st);
    launch_finalize_slots(sl.partials, 0, c->d, np, false, io[si].isc + I_SUMV, st);
  }
  comm_allreduce(c, intls(io, I_SUMV), c->d, false, st);
  if (P > 1) {  // SL-step inputs: max |delta_z| over both feet
    window_of(window_decision(c, [](Slab& s) { return (const float*)s.df + 2 * s.F; },
                              want_adj ? std::function<const float*(Slab&)>([](Slab& s) { return (const float*)s.da + 2 * s.F; })
                                       : std::function<const float*(Slab&)>(),
                              1, st),
              c->zw_m, c->wrap_m);
  }
  const int zw = c->zw_m;
  const bool cont = c->p.model == TOPT_CONTINUITY;
  if (cont) {
    if (c->div_pending) {
      cudaStreamWaitEvent(st, c->ev_div, 0);
      c->div_pending = false;
    } else {
      Prof pr(c, K_DIV, (3.0 * d - 1.0) * F4, c->d, st);
      compute_div(c, io, st);
    }
    if (zw) sl_input(c, [](Slab& s) { return s.divv; }, 1, 0, zw, st);
    for (auto& sl : c->slabs) {
      Prof pr(c, K_EFACTOR, (d + 2) * F4, 1, st);
      launch_efactor(in_geom(c, sl, zw, c->wrap_m), in_ptr(sl, sl.divv, zw), sl.df, (float)(-0.5 * c->dt),
                     (float)(0.5 * c->dt * c->dt), sl.E, st);
    }
  }
  const double e = cont ? 1.0 : 0.0;
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    Prof pr(c, K_MISC, 2.0 * F4, 0, st);
    cudaMemcpyAsync(local(sl, sl.m_traj), io[si].m0, sl.F * 4, cudaMemcpyDeviceToDevice, st);
  }
  std::vector<int> np(c->slabs.size(), 0);
  for (int j = 0; j < S; ++j) {
    sl_input(c, [j](Slab& s) { return s.m_traj + j * s.Fh; }, 1, 0, zw, st);
    for (size_t si = 0; si < c->slabs.size(); ++si) {
      Slab& sl = c->slabs[si];
      const float* Ef = cont ? sl.E : nullptr;
      const Geom gi = in_geom(c, sl, zw, c->wrap_m);
      const float* in = in_ptr(sl, sl.m_traj + j * sl.Fh, zw);
      if (j + 1 < S) {
        Prof pr(c, K_SL_STEP, (d + 2 + e) * F4, 1, st);
        launch_sl_step(gi, in, sl.df, Ef, local(sl, sl.m_traj + (j + 1) * sl.Fh), st);
      } else {
        Prof pr(c, K_SL_LAST, (d + 4 + e) * F4, 1, st);
        launch_sl_last(gi, in, sl.df, Ef, io[si].m1, local(sl, sl.m_traj + S * sl.Fh),
                       local(sl, sl.lam_traj + S * sl.Fh), sl.partials, &np[si], st);
      }
    }
  }
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Prof pr(c, K_MISC, 0.0, 1, st);
    launch_finalize(c->slabs[si].partials, 0, np[si], 0.5 * c->cellvol, false, io[si].scal + TOPT_S_DIST, st);
  }
  comm_allreduce(c, pubs(io, TOPT_S_DIST), 1, false, st);
}

// Backward half: adjoint sweep (advection: Heun factor, R7), body force (2.2)/(R8) with
// trapezoid weights (R10), then g = alpha L v + b (P_L b for incompressible, R9) and
// s = -(alpha L~)^{-1} g = -P_0 v - (alpha L~)^{-1} b.  alpha L v is `u` when the
// caller tracks it (solver), otherwise computed by the fp64 v-chain into utmp.
void backward_half(topt_ctx* c, std::vector<Io>& io, cudaStream_t st) {
  const int S = c->p.nt, P = P_of(c);
  const size_t F = c->F;
  const double F4 = 4.0 * F, d = c->d;
  const bool adv = c->p.model == TOPT_ADVECTION;
  const int zw = c->zw_m;  // sized by forward_half from both feet
  if (adv) {
    if (c->div_pending) {
      cudaStreamWaitEvent(st, c->ev_div, 0);
      c->div_pending = false;
    } else {
      Prof pr(c, K_DIV, (3.0 * d - 1.0) * F4, c->d, st);
      compute_div(c, io, st);
    }
    if (zw) sl_input(c, [](Slab& s) { return s.divv; }, 1, 0, zw, st);
    for (auto& sl : c->slabs) {
      Prof pr(c, K_EFACTOR, (d + 2) * F4, 1, st);
      launch_efactor(in_geom(c, sl, zw, c->wrap_m), in_ptr(sl, sl.divv, zw), sl.da, (float)(0.5 * c->dt),
                     (float)(0.5 * c->dt * c->dt), sl.E, st);
    }
  }
  const double e = adv ? 1.0 : 0.0;
  for (int j = S - 1; j >= 0; --j) {
    sl_input(c, [j](Slab& s) { return s.lam_traj + (j + 1) * s.Fh; }, 1, 0, zw, st);
    for (auto& sl : c->slabs) {
      Prof pr(c, K_SL_STEP, (d + 2 + e) * F4, 1, st);
      launch_sl_step(in_geom(c, sl, zw, c->wrap_m), in_ptr(sl, sl.lam_traj + (j + 1) * sl.Fh, zw), sl.da,
                     adv ? sl.E : nullptr, local(sl, sl.lam_traj + j * sl.Fh), st);
    }
  }
  // body force
  std::vector<double> w = c->wts;
  const bool cont = c->p.model == TOPT_CONTINUITY;
  if (cont)
    for (auto& x : w) x = -x;
  const int nloc_axes = P > 1 ? 2 : c->d;
  for (auto& sl : c->slabs) {
    float* psi = local(sl, cont ? sl.lam_traj : sl.m_traj);
    float* lam = local(sl, cont ? sl.m_traj : sl.lam_traj);
    for (int a = 0; a < nloc_axes; ++a) {
      Prof pr(c, K_BODY, (2.0 * (S + 1) + 1.0) * F4, 1, st);
      DerivArgs da{psi, sl.Fh, lam, sl.Fh, w.data(), S + 1, 0.f, sl.b + a * F};
      launch_deriv_accum(sl.g, a, da, st);
    }
  }
  if (P > 1 && comm_p2p_ready(c)) {
    // z axis, P2P transport: one kernel per rank reads the z-lines of its y rows from every
    // rank's slices and writes b_z into every rank's slab (transposes fused away)
    comm_fence(c, st);  // every rank's trajectories are complete
    const bool emu = c->comm.emulated();
    for (auto& sl : c->slabs) {
      const float *ps[8], *ls[8];
      float* os[8];
      for (int q = 0; q < P; ++q) {
        Slab& sq = emu ? c->slabs[q] : c->slabs[0];  // one process per GPU: peers by translation
        ps[q] = (const float*)comm_peer(c, local(sq, cont ? sq.lam_traj : sq.m_traj), q);
        ls[q] = (const float*)comm_peer(c, local(sq, cont ? sq.m_traj : sq.lam_traj), q);
        os[q] = (float*)comm_peer(c, sq.b + 2 * F, q);
      }
      Prof pr(c, K_BODY, (2.0 * (S + 1) + 1.0) * F4, 1, st);
      launch_deriv_zpull(sl.gy, ps, ls, os, P, sl.Fh, sl.Fh, sl.g.nz, sl.plane, w.data(), S + 1, st);
    }
    comm_fence(c, st);  // every rank's b_z is complete before it is read
  } else if (P > 1) {  // z axis in the y-slab layout: transpose all S+1 slices of psi and lam
    for (int j = 0; j <= S; ++j)
      for (int which = 0; which < 2; ++which) {  // 0: psi, 1: lam
        std::vector<float*> src, dst;
        for (auto& sl : c->slabs) {
          float* traj = ((which == 0) == cont) ? sl.lam_traj : sl.m_traj;
          src.push_back(local(sl, traj + j * sl.Fh));
          dst.push_back(sl.ytraj + ((size_t)which * (S + 1) + j) * F);
        }
        tz2y(c, src, dst, st);
      }
    std::vector<float*> ysrc, zdst;
    for (auto& sl : c->slabs) {
      Prof pr(c, K_BODY, (2.0 * (S + 1) + 1.0) * F4, 1, st);
      DerivArgs da{sl.ytraj, F, sl.ytraj + (S + 1) * F, F, w.data(), S + 1, 0.f, sl.ytmp};
      launch_deriv_accum(sl.gy, 2, da, st);
      ysrc.push_back(sl.ytmp);
      zdst.push_back(sl.b + 2 * F);
    }
    ty2z(c, ysrc, zdst, st);
  }
  const bool leray = c->p.model == TOPT_INCOMPRESSIBLE;
  const double half = c->d == 3 ? 2.0 : 1.0;
  const double n_all = ntot(c);
  if (merged_chain(c, io)) {
    if (c->vf_pending) {
      cudaStreamWaitEvent(st, c->ev_u, 0);
      c->vf_pending = false;
    } else {
      vchain_fwd(c, io, st);
    }
    Slab& sl = c->slabs[0];
    const double F8 = 8.0 * F, F16 = 16.0 * F, half = c->d == 3 ? 2.0 : 1.0;
    float2* Z[4] = {sl.Z, sl.Z + F, sl.Z + 2 * F, sl.Z + 3 * F};
    double2* Zv[3] = {sl.Zv, sl.Zv + F, sl.Zv + 2 * F};
    int npz = 0;
    {
      const double bytes = d * F4 + half * F8 + (c->d == 3 ? 2 * half * F8 : 0.0) +       // b x, y forward
                           half * (F16 + F8) + 2 * half * F8 +                                 // merged last axis
                           (c->d == 3 ? 2 * 2 * half * F8 : 0.0);                            // y^-1 of g^, p^
      Prof pr(c, K_BCHAIN, bytes, c->d == 3 ? 4 : 2, st);
      bchain_xy(sl.g, sl.b, Z, false, st);
      gchain_last(sl.g, Zv, Z, c->p.alpha, c->p.reg_order, (double)F, sl.partials, &npz, st);
      gchain_yinv(sl.g, Z, st);
    }
    int np = 0;
    {
      Prof pr(c, K_ASSEMBLE, 2 * half * F8 + d * F4 + 2 * d * F4, 1, st);
      launch_assemble(sl.g, sl.Z, true, nullptr, nullptr, io[0].v, io[0].isc + I_SUMV, io[0].g, io[0].s,
                      sl.partials, &np, st, (double)F);
    }
    {
      Prof pr(c, K_MISC, 0.0, 1, st);
      launch_finalize_slots(sl.partials, 0, 10, np, true, io[0].isc + I_GMAX, st);
      // v.u and s.u from the merged pass (slots 10, 11), unnormalised spectra: / n
      launch_finalize_multi_k(sl.partials, 10, 2, npz, 1.0 / (double)F, io[0].isc + I_VU, st);
    }
    launch_finish(io[0].isc, io[0].scal, c->d, (double)F, c->cellvol, st);
    return;
  }
  // v-chain: u = alpha L v (fp64) when not supplied (or already running on the side stream)
  if (c->u_pending) {
    cudaStreamWaitEvent(st, c->ev_u, 0);
    c->u_pending = false;
    for (size_t si = 0; si < c->slabs.size(); ++si) io[si].u = c->slabs[si].utmp;
  } else if (io[0].u == nullptr) {
    run_vchain(c, io, st);
  }
  {
    const double nin = leray ? d : half, nout = leray ? 2 * half : half, F8 = 8.0 * F;
    const double bytes = d * F4 + nin * F8 + (c->d == 3 ? 2 * nin * F8 + 2 * nout * F8 : 0.0) + (nin + nout) * F8;
    Prof pr(c, K_BCHAIN, bytes * c->comm.nloc, c->d == 3 ? 4 : 2, st);
    const int bin = bchain_nin(c->slabs[0].g, leray), bout = bchain_nout(c->slabs[0].g, leray);
    for (auto& sl : c->slabs) {
      float2* Z[4] = {sl.Z, sl.Z + F, sl.Z + 2 * F, sl.Z + 3 * F};
      bchain_xy(sl.g, sl.b, Z, leray, st);
    }
    std::vector<const void*> rtab;
    if (remote_fields<float2>(c, [](Slab& s) { return s.Z; }, bin, rtab)) {
      comm_fence(c, st);
      for (auto& sl : c->slabs)
        bchain_last_remote(sl.gy, rtab.data(), P, sl.g.nz, sl.plane, c->p.alpha, c->p.reg_order, n_all, st);
      comm_fence(c, st);
    } else {
      if (P > 1)
        for (int f = 0; f < bin; ++f) {
          std::vector<float2*> a, b;
          for (auto& sl : c->slabs) { a.push_back(sl.Z + f * F); b.push_back(sl.Zy + f * F); }
          tz2y(c, a, b, st);
        }
      for (auto& sl : c->slabs) {
        float2* base = P > 1 ? sl.Zy : sl.Z;
        float2* Z[4] = {base, base + F, base + 2 * F, base + 3 * F};
        bchain_last(P > 1 ? sl.gy : sl.g, Z, c->p.alpha, c->p.reg_order, leray, n_all, st);
      }
      if (P > 1)
        for (int f = 0; f < bout; ++f) {
          std::vector<float2*> a, b;
          for (auto& sl : c->slabs) { a.push_back(sl.Zy + f * F); b.push_back(sl.Z + f * F); }
          ty2z(c, a, b, st);
        }
    }
    for (auto& sl : c->slabs) {
      float2* Z[4] = {sl.Z, sl.Z + F, sl.Z + 2 * F, sl.Z + 3 * F};
      bchain_yinv(sl.g, Z, leray, st);
    }
  }
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    int np = 0;
    {
      const double nout = leray ? 2 * half : half;
      const double bytes = nout * 8.0 * F + (leray ? 0.0 : d * F4) + 2 * d * F4 + 2 * d * F4;
      Prof pr(c, K_ASSEMBLE, bytes, 1, st);
      launch_assemble(sl.g, sl.Z, leray, sl.b, io[si].u, io[si].v, io[si].isc + I_SUMV, io[si].g, io[si].s,
                      sl.partials, &np, st, n_all);
    }
    Prof pr(c, K_MISC, 0.0, 1, st);
    launch_finalize_slots(sl.partials, 0, 10, np, true, io[si].isc + I_GMAX, st);
  }
  comm_allreduce(c, intls(io, I_GMAX), 1, true, st);
  comm_allreduce(c, intls(io, I_GS), I_SUMS + 3 - I_GS, false, st);
  for (size_t si = 0; si < c->slabs.size(); ++si) launch_finish(io[si].isc, io[si].scal, c->d, n_all, c->cellvol, st);
}

// One objective + gradient evaluation.  On a single slab, div v and the fp64 v-chain
// depend on v alone: they run on the library's side stream (forked from and joined back
// into `st` by events) concurrently with the trace and the SL sweeps, which are bound by
// shared memory and leave most of the HBM bandwidth idle.  With z-slabs (NCCL exchanges
// inside both) everything stays on `st`.
topt_status eval_gradient(topt_ctx* c, std::vector<Io>& io, cudaStream_t st) {
  c->div_pending = c->u_pending = c->vf_pending = false;
  // (profiling mode serialises everything on `st`, so the per-class times are standalone)
  if (P_of(c) == 1 && c->side && io[0].u == nullptr && !c->prof) {
    cudaEventRecord(c->ev_fork, st);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    if (c->p.model != TOPT_INCOMPRESSIBLE) {
      {
        Prof pr(c, K_DIV, (3.0 * c->d - 1.0) * 4.0 * c->F, c->d, c->side);
        compute_div(c, io, c->side);
      }
      cudaEventRecord(c->ev_div, c->side);
      c->div_pending = true;
    }
    if (merged_chain(c, io)) {  // only the fp64 forward passes of v are independent of b
      vchain_fwd(c, io, c->side);
      c->vf_pending = true;
    } else {
      run_vchain(c, io, c->side);
      for (auto& x : io) x.u = nullptr;  // set again when the v-chain is joined
      c->u_pending = true;
    }
    cudaEventRecord(c->ev_u, c->side);
  }
  forward_half(c, io, true, st);
  backward_half(c, io, st);
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

// Copy a scalar set to the host; with z-slabs also the halo-overflow flag, all-reduced (max)
// over every slab so that all ranks take the same decision.
topt_status fetch(topt_ctx* c, int set, HostScalars& out, cudaStream_t st) {
  if (c->comm.P > 1) {
    std::vector<double*> fl;
    for (auto& sl : c->slabs) {
      double* slot = sl.sc + set * kSet + kSet - 1;
      launch_flag_to_double(sl.haloerr, slot, st);
      fl.push_back(slot);
    }
    comm_allreduce(c, fl, 1, true, st);
  }
  TOPT_CUDA(cudaMemcpyAsync(out.v, c->slabs[0].sc + set * kSet, sizeof(out.v), cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  if (c->comm.P > 1 && out.v[kSet - 1] != 0.0)
    return fail(TOPT_ERR_HALO, "internal: a characteristic foot left the sized z-slab window");
  return TOPT_OK;
}

// dots[i] = <a, bs[i]> (unweighted l2 over all d*n entries of all slabs), on the host.
topt_status host_dots(topt_ctx* c, std::function<const float*(Slab&)> a,
                      const std::vector<std::function<const float*(Slab&)>>& bs, std::vector<double>& out,
                      cudaStream_t st) {
  const int n = (int)bs.size();
  out.assign(n, 0.0);
  if (n == 0) return TOPT_OK;
  std::vector<double*> dd;
  for (auto& sl : c->slabs) {
    std::vector<const float*> b;
    for (auto& f : bs) b.push_back(f(sl));
    int np = 0;
    {
      Prof pr(c, K_GRAM, (n + 1.0) * c->vecN * 4.0, 1, st);  // a and every b read once (a8)
      launch_multidot(a(sl), b.data(), n, c->vecN, sl.partials, &np, st);
    }
    launch_finalize_multi(sl.partials, 0, n, np, 1.0, sl.dots, st);
    dd.push_back(sl.dots);
  }
  comm_allreduce(c, dd, n, false, st);
  TOPT_CHECK_LAUNCH();
  TOPT_CUDA(cudaMemcpyAsync(out.data(), c->slabs[0].dots, n * 8, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

// in-place Leray projection of a per-slab vector field (b-chain with b := x; assemble -> P_L x)
void leray_inplace(topt_ctx* c, std::function<float*(Slab&)> x, cudaStream_t st) {
  const int P = P_of(c);
  const size_t F = c->F;
  const int bin = bchain_nin(c->slabs[0].g, true), bout = bchain_nout(c->slabs[0].g, true);
  for (auto& sl : c->slabs) {
    float2* Z[4] = {sl.Z, sl.Z + F, sl.Z + 2 * F, sl.Z + 3 * F};
    bchain_xy(sl.g, x(sl), Z, true, st);
  }
  if (P > 1)
    for (int f = 0; f < bin; ++f) {
      std::vector<float2*> a, b;
      for (auto& sl : c->slabs) { a.push_back(sl.Z + f * F); b.push_back(sl.Zy + f * F); }
      tz2y(c, a, b, st);
    }
  for (auto& sl : c->slabs) {
    float2* base = P > 1 ? sl.Zy : sl.Z;
    float2* Z[4] = {base, base + F, base + 2 * F, base + 3 * F};
    bchain_last(P > 1 ? sl.gy : sl.g, Z, c->p.alpha, c->p.reg_order, true, ntot(c), st);
  }
  if (P > 1)
    for (int f = 0; f < bout; ++f) {
      std::vector<float2*> a, b;
      for (auto& sl : c->slabs) { a.push_back(sl.Zy + f * F); b.push_back(sl.Z + f * F); }
      ty2z(c, a, b, st);
    }
  for (auto& sl : c->slabs) {
    float2* Z[4] = {sl.Z, sl.Z + F, sl.Z + 2 * F, sl.Z + 3 * F};
    bchain_yinv(sl.g, Z, true, st);
    int np = 0;
    launch_assemble(sl.g, sl.Z, true, nullptr, nullptr, nullptr, nullptr, x(sl), nullptr, sl.partials, &np, st);
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Emulated z-slabs: the caller passes whole-grid arrays; slab s of a scalar field is the
// contiguous block s*F, of component c of a vector field the block c*F_all + s*F.
bool emu(const topt_ctx* c) { return c->comm.P > 1 && c->comm.emulated(); }

void stage_vec_in(topt_ctx* c, const float* full, std::function<float*(Slab&)> dst, cudaStream_t st) {
  const size_t F = c->F, Fall = F * c->comm.P;
  for (size_t si = 0; si < c->slabs.size(); ++si)
    for (int a = 0; a < c->d; ++a)
      cudaMemcpyAsync(dst(c->slabs[si]) + a * F, full + a * Fall + si * F, F * 4, cudaMemcpyDeviceToDevice, st);
}
void stage_vec_out(topt_ctx* c, std::function<const float*(Slab&)> src, float* full, cudaStream_t st) {
  const size_t F = c->F, Fall = F * c->comm.P;
  for (size_t si = 0; si < c->slabs.size(); ++si)
    for (int a = 0; a < c->d; ++a)
      cudaMemcpyAsync(full + a * Fall + si * F, src(c->slabs[si]) + a * F, F * 4, cudaMemcpyDeviceToDevice, st);
}

// Build the per-slab Io of an evaluation at user pointers (emulation: staged copies).
std::vector<Io> make_io(topt_ctx* c, const float* m0, const float* m1, const float* v, int set, cudaStream_t st) {
  std::vector<Io> io(c->slabs.size());
  if (emu(c)) stage_vec_in(c, v, [](Slab& s) { return s.vb; }, st);
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    io[si].m0 = emu(c) ? m0 + si * sl.F : m0;
    io[si].m1 = emu(c) ? m1 + si * sl.F : m1;
    io[si].v = emu(c) ? sl.vb : v;
    io[si].u = nullptr;
    io[si].g = sl.gcur;
    io[si].s = sl.scur;
    io[si].scal = sl.pub(set);
    io[si].isc = sl.intl(set);
  }
  return io;
}

}  // namespace

// ======================================================================================
// ABI entry points
// ======================================================================================
extern "C" {

// Replay a captured evaluation for this pointer key, capturing it on first use: the work
// `body(stream)` is recorded on the library's capture stream (the caller's stream may be the
// legacy default stream, which cannot capture), instantiated once and launched on `st`.
// One slab only (no host decisions, no collectives); profiling mode runs eagerly.
static bool graphs_ok(topt_ctx* c) { return c->use_graphs && !c->prof && c->comm.P == 1; }
static topt_status graph_run(topt_ctx* c, const void* const key[8], cudaStream_t st,
                             const std::function<topt_status(cudaStream_t)>& body) {
  for (auto& ge : c->graphs)
    if (std::equal(ge.key, ge.key + 8, key)) {
      TOPT_CUDA(cudaGraphLaunch(ge.exec, st));
      launch_count_add(ge.nlaunch);
      return TOPT_OK;
    }
  if (!c->gcap) {
    TOPT_CUDA(cudaStreamCreateWithFlags(&c->gcap, cudaStreamNonBlocking));
    TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_gcap, cudaEventDisableTiming));
  }
  const long long l0 = launch_count();
  TOPT_CUDA(cudaStreamBeginCapture(c->gcap, cudaStreamCaptureModeRelaxed));
  topt_status r = body(c->gcap);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->gcap, &graph);
  if (r != TOPT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  if (ec != cudaSuccess) return fail(TOPT_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return fail(TOPT_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
  topt_ctx::GraphEntry ge;
  std::copy(key, key + 8, ge.key);
  ge.exec = exec;
  ge.nlaunch = launch_count() - l0;
  launch_count_add(-ge.nlaunch);  // captured, not launched
  if ((int)c->graphs.size() >= kMaxGraphs) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back(ge);
  TOPT_CUDA(cudaGraphLaunch(exec, st));
  launch_count_add(ge.nlaunch);
  return TOPT_OK;
}

// z-slab evaluation (P > 1) through segmented graphs: replay segment k, read window decision k,
// pick segment k+1 by it.  A missing segment re-runs the evaluation's host code under capture from
// the start, reusing the decisions of the segments this evaluation already launched (those are
// only re-cached).  NCCL collectives and point-to-point calls are captured like kernels.  A failed
// capture switches slab graphs off for the context and the evaluation is re-run eagerly.
static bool slab_graphs_ok(topt_ctx* c) { return c->use_graphs && !c->prof && c->comm.P > 1 && !c->slab_graphs_off; }
static topt_status eval_slab_graphs(topt_ctx* c, std::vector<Io>& io, const void* const base[6], cudaStream_t st) {
  std::vector<int> dec;
  for (int seg = 0; seg < kSlabSegs; ++seg) {
    const void* key[8];
    seg_key(key, base, seg, dec);
    topt_ctx::GraphEntry* ge = find_graph(c, key);
    if (!ge) break;
    TOPT_CUDA(cudaGraphLaunch(ge->exec, st));
    launch_count_add(ge->nlaunch);
    if (seg + 1 == kSlabSegs) {
      window_of(dec[0], c->zw_v, c->wrap_v);
      window_of(dec[1], c->zw_m, c->wrap_m);
      return TOPT_OK;
    }
    dec.push_back(decision_of(c, zmax_read(c, st), seg));
  }
  if (!c->gcap) {
    TOPT_CUDA(cudaStreamCreateWithFlags(&c->gcap, cudaStreamNonBlocking));
    TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_gcap, cudaEventDisableTiming));
  }
  topt_ctx::SegCap& sc = c->segc;
  sc.err = false;
  sc.user = st;
  std::copy(base, base + 6, sc.base);
  sc.known = dec;
  sc.dec.clear();
  sc.l0 = launch_count();
  c->div_pending = c->u_pending = c->vf_pending = false;
  if (cudaStreamBeginCapture(c->gcap, cudaStreamCaptureModeRelaxed) != cudaSuccess) sc.err = true;
  if (!sc.err) {
    sc.on = true;
    forward_half(c, io, true, c->gcap);
    backward_half(c, io, c->gcap);
    if (!sc.err) seg_end(c, true, true);
    sc.on = false;
  }
  if (!sc.err) return TOPT_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->gcap, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
    cudaGraph_t gr = nullptr;
    cudaStreamEndCapture(c->gcap, &gr);
    if (gr) cudaGraphDestroy(gr);
  }
  cudaStreamSynchronize(c->gcap);
  cudaGetLastError();
  c->slab_graphs_off = true;
  return eval_gradient(c, io, st);
}

topt_status topt_eval_gradient(topt_ctx* c, const float* m0, const float* m1, const float* v, float* g, float* s,
                               double* d_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (!aligned16(m0) || !aligned16(m1) || !aligned16(v) || (g && !aligned16(g)) || (s && !aligned16(s)))
    return fail(TOPT_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (graphs_ok(c)) {
    const void* key[8] = {(const void*)1, m0, m1, v, g, s, d_scalars, nullptr};
    return graph_run(c, key, st, [&](cudaStream_t cs) -> topt_status {
      std::vector<Io> io = make_io(c, m0, m1, v, 4, cs);
      io[0].g = g;
      io[0].s = s;
      io[0].scal = d_scalars;
      topt_status rr = eval_gradient(c, io, cs);
      TOPT_CHECK_LAUNCH();
      return rr;
    });
  }
  std::vector<Io> io = make_io(c, m0, m1, v, 4, st);
  if (!emu(c)) {
    io[0].g = g;
    io[0].s = s;
    io[0].scal = d_scalars;
  }
  const void* base[6] = {m0, m1, v, g, s, d_scalars};
  topt_status r = slab_graphs_ok(c) ? eval_slab_graphs(c, io, base, st) : eval_gradient(c, io, st);
  if (r != TOPT_OK) return r;
  if (emu(c)) {
    if (g) stage_vec_out(c, [](Slab& x) { return (const float*)x.gcur; }, g, st);
    if (s) stage_vec_out(c, [](Slab& x) { return (const float*)x.scur; }, s, st);
    TOPT_CUDA(cudaMemcpyAsync(d_scalars, c->slabs[0].pub(4), TOPT_NSCALARS * 8, cudaMemcpyDeviceToDevice, st));
  }
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_eval_gradient_host(topt_ctx* c, const float* m0_h, const float* m1_h, const float* v_h, float* g_h,
                                    double* h_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0_h || !m1_h || !v_h || !h_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (emu(c)) return fail(TOPT_ERR_UNSUPPORTED, "host-buffer evaluation with emulated slabs");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  TOPT_CUDA(cudaMemcpyAsync(sl.m0b, m0_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(sl.m1b, m1_h, c->F * 4, cudaMemcpyHostToDevice, st));
  TOPT_CUDA(cudaMemcpyAsync(sl.vb, v_h, c->vecN * 4, cudaMemcpyHostToDevice, st));
  std::vector<Io> io = make_io(c, sl.m0b, sl.m1b, sl.vb, 4, st);
  topt_status r = eval_gradient(c, io, st);
  if (r != TOPT_OK) return r;
  if (g_h) TOPT_CUDA(cudaMemcpyAsync(g_h, sl.gcur, c->vecN * 4, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaMemcpyAsync(h_scalars, sl.pub(4), TOPT_NSCALARS * 8, cudaMemcpyDeviceToHost, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
  return TOPT_OK;
}

// Two staging slots: slot 0 = (m0b, m1b, vb) -> (gcur, scur, scalar set 4), slot 1 =
// (q[0, F), q[F, 2F), vt) -> (gq, sq, set 3) (solver vectors, idle outside topt_solve).
// Per call, slot b:  h_in: wait free[b]; H2D; record in[b]  |  h_comp: wait in[b], out[b];
// evaluate; record free[b], done[b]  |  h_out: wait done[b]; D2H; record out[b]  |
// caller stream: wait out[b].
topt_status topt_eval_gradient_host_async(topt_ctx* c, const float* m0_h, const float* m1_h, const float* v_h,
                                          float* g_h, double* h_scalars, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0_h || !m1_h || !v_h || !h_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (P_of(c) != 1) return fail(TOPT_ERR_UNSUPPORTED, "streaming host evaluation needs world == 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->h_in) {
    TOPT_CUDA(cudaStreamCreateWithFlags(&c->h_in, cudaStreamNonBlocking));
    TOPT_CUDA(cudaStreamCreateWithFlags(&c->h_comp, cudaStreamNonBlocking));
    TOPT_CUDA(cudaStreamCreateWithFlags(&c->h_out, cudaStreamNonBlocking));
    TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_hfork, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_hin[i], cudaEventDisableTiming));
      TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_hfree[i], cudaEventDisableTiming));
      TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_hdone[i], cudaEventDisableTiming));
      TOPT_CUDA(cudaEventCreateWithFlags(&c->ev_hout[i], cudaEventDisableTiming));
    }
  }
  const int b = c->hslot;
  c->hslot ^= 1;
  Slab& sl = c->slabs[0];
  float* m0d = b ? sl.q : sl.m0b;
  float* m1d = b ? sl.q + sl.F : sl.m1b;
  float* vd = b ? sl.vt : sl.vb;
  const int set = b ? 3 : 4;
  // the inputs are host buffers: the copy-in does not wait for earlier work on `stream`
  // (which, after a previous call, ends with that call's copy-out), only for the slot
  TOPT_CUDA(cudaStreamWaitEvent(c->h_in, c->ev_hfree[b], 0));
  TOPT_CUDA(cudaMemcpyAsync(m0d, m0_h, c->F * 4, cudaMemcpyHostToDevice, c->h_in));
  TOPT_CUDA(cudaMemcpyAsync(m1d, m1_h, c->F * 4, cudaMemcpyHostToDevice, c->h_in));
  TOPT_CUDA(cudaMemcpyAsync(vd, v_h, c->vecN * 4, cudaMemcpyHostToDevice, c->h_in));
  TOPT_CUDA(cudaEventRecord(c->ev_hin[b], c->h_in));
  TOPT_CUDA(cudaStreamWaitEvent(c->h_comp, c->ev_hin[b], 0));
  TOPT_CUDA(cudaStreamWaitEvent(c->h_comp, c->ev_hout[b], 0));
  float* gd = b ? sl.gq : sl.gcur;
  float* sd = b ? sl.sq : sl.scur;
  auto body = [&](cudaStream_t cs) -> topt_status {
    std::vector<Io> io = make_io(c, m0d, m1d, vd, set, cs);
    io[0].g = gd;
    io[0].s = sd;
    return eval_gradient(c, io, cs);
  };
  const void* key[8] = {(const void*)2, m0d, m1d, vd, gd, sd, sl.pub(set), nullptr};
  topt_status r = graphs_ok(c) ? graph_run(c, key, c->h_comp, body) : body(c->h_comp);
  if (r != TOPT_OK) return r;
  TOPT_CUDA(cudaEventRecord(c->ev_hfree[b], c->h_comp));
  TOPT_CUDA(cudaEventRecord(c->ev_hdone[b], c->h_comp));
  TOPT_CUDA(cudaStreamWaitEvent(c->h_out, c->ev_hdone[b], 0));
  if (g_h) TOPT_CUDA(cudaMemcpyAsync(g_h, gd, c->vecN * 4, cudaMemcpyDeviceToHost, c->h_out));
  TOPT_CUDA(cudaMemcpyAsync(h_scalars, sl.pub(set), TOPT_NSCALARS * 8, cudaMemcpyDeviceToHost, c->h_out));
  TOPT_CUDA(cudaEventRecord(c->ev_hout[b], c->h_out));
  TOPT_CUDA(cudaStreamWaitEvent(st, c->ev_hout[b], 0));
  return TOPT_OK;
}

topt_status topt_objective(topt_ctx* c, const float* m0, const float* m1, const float* v, double* d_scalars,
                           void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !m1 || !v || !d_scalars) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<Io> io = make_io(c, m0, m1, v, 4, st);
  forward_half(c, io, false, st);
  // reg = alpha/2 <v, L v>_h = h^d/2 sum v u,  u = alpha L v (fp64 chain, plain L as in (1.1a))
  const int P = P_of(c);
  const size_t F = c->F;
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    double2* Z[3] = {sl.Zv, sl.Zv + F, sl.Zv + 2 * F};
    vchain_xy(sl.g, io[si].v, Z, false, st);
  }
  const int vin = vchain_nin(c->slabs[0].g, false), vout = vchain_nout(c->slabs[0].g);
  if (P > 1)
    for (int f = 0; f < vin; ++f) {
      std::vector<double2*> a, b;
      for (auto& sl : c->slabs) { a.push_back(sl.Zv + f * F); b.push_back(sl.Zvy + f * F); }
      tz2y(c, a, b, st);
    }
  for (auto& sl : c->slabs) {
    double2* base = P > 1 ? sl.Zvy : sl.Zv;
    double2* Z[3] = {base, base + F, base + 2 * F};
    vchain_last(P > 1 ? sl.gy : sl.g, Z, c->p.alpha, c->p.reg_order, false, ntot(c), st);
  }
  if (P > 1)
    for (int f = 0; f < vout; ++f) {
      std::vector<double2*> a, b;
      for (auto& sl : c->slabs) { a.push_back(sl.Zvy + f * F); b.push_back(sl.Zv + f * F); }
      ty2z(c, a, b, st);
    }
  std::vector<double*> regs;
  for (size_t si = 0; si < c->slabs.size(); ++si) {
    Slab& sl = c->slabs[si];
    double2* Z[3] = {sl.Zv, sl.Zv + F, sl.Zv + 2 * F};
    vchain_inv(sl.g, Z, sl.utmp, st);
    const float* bs[1] = {sl.utmp};
    int np = 0;
    launch_multidot(io[si].v, bs, 1, c->vecN, sl.partials, &np, st);
    launch_finalize_multi(sl.partials, 0, 1, np, 0.5 * c->cellvol, io[si].scal + TOPT_S_REG, st);
    regs.push_back(io[si].scal + TOPT_S_REG);
  }
  comm_allreduce(c, regs, 1, false, st);
  for (auto& x : io) launch_combine_obj(x.scal, st);
  TOPT_CUDA(cudaMemcpyAsync(d_scalars, io[0].scal, TOPT_NSCALARS * 8, cudaMemcpyDeviceToDevice, st));
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

static topt_status single_slab(topt_ctx* c) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (c->comm.P != 1) return fail(TOPT_ERR_UNSUPPORTED, "per-operator entry points run on one slab (world == 1)");
  return TOPT_OK;
}

topt_status topt_feet(topt_ctx* c, const float* v, float* delta_f, float* delta_a, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!v || (!delta_f && !delta_a)) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  launch_trace(c->slabs[0].g, v, delta_f, delta_a, nullptr, nullptr, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_forward(topt_ctx* c, const float* m0, const float* v, float* m_traj, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!m0 || !v || !m_traj) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<Io> io = make_io(c, m0, m0, v, 4, st);
  forward_half(c, io, false, st);
  TOPT_CUDA(cudaMemcpyAsync(m_traj, c->slabs[0].m_traj, (c->p.nt + 1) * c->F * 4, cudaMemcpyDeviceToDevice, st));
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_get_adjoint(topt_ctx* c, float* lam_traj, float* body_force, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  cudaStream_t st = (cudaStream_t)stream;
  if (lam_traj)
    TOPT_CUDA(cudaMemcpyAsync(lam_traj, c->slabs[0].lam_traj, (c->p.nt + 1) * c->F * 4, cudaMemcpyDeviceToDevice,
                              st));
  if (body_force) TOPT_CUDA(cudaMemcpyAsync(body_force, c->slabs[0].b, c->vecN * 4, cudaMemcpyDeviceToDevice, st));
  return TOPT_OK;
}

topt_status topt_derivative(topt_ctx* c, const float* f, int32_t axis, float* out, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!f || !out) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  if (axis < 0 || axis >= c->d) return fail(TOPT_ERR_INVALID_ARG, "axis out of range");
  double one = 1.0;
  DerivArgs da{f, 0, nullptr, 0, &one, 1, 0.f, out};
  launch_deriv_accum(c->slabs[0].g, axis, da, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

// Flow map y and det(grad y) (figure captions; reading R32): the
// displacement u = y - x is composed over the n_t backward SL maps with the static RK2
// foot, u^{j+1} = delta_f + I[u^j](l + delta_f); J[b][a] = d_a (h_b u_b) by the spectral
// derivative kernels; det(I + J) pointwise (fp64 arithmetic on fp32 J).
topt_status topt_flow_map(topt_ctx* c, const float* v, float* y_disp, float* det, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!v || !y_disp || !det) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  const int d = c->d, S = c->p.nt;
  launch_trace(sl.g, v, sl.df, nullptr, nullptr, nullptr, st);
  float* ua = sl.utmp;
  float* ub = sl.b;
  TOPT_CUDA(cudaMemsetAsync(ua, 0, c->vecN * 4, st));
  for (int j = 0; j < S; ++j) {
    launch_flow_step(sl.g, ua, sl.df, ub, st);
    std::swap(ua, ub);
  }
  float* J = reinterpret_cast<float*>(sl.Zv);  // d*d fields of F (Zv holds 12 F floats)
  for (int b = 0; b < d; ++b)
    for (int a = 0; a < d; ++a) {
      const double hb = c->h[b];
      DerivArgs da{ua + (size_t)b * sl.F, 0, nullptr, 0, &hb, 1, 0.f, J + (size_t)(b * d + a) * sl.F};
      launch_deriv_accum(sl.g, a, da, st);
    }
  launch_flow_det(sl.g, ua, J, c->h, y_disp, det, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_apply_precond(topt_ctx* c, const float* g, float* s, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!g || !s) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  const bool leray = c->p.model == TOPT_INCOMPRESSIBLE;
  launch_bchain(sl.g, g, sl.Z, c->p.alpha, c->p.reg_order, leray, st);
  int np = 0;
  launch_assemble(sl.g, sl.Z, leray, g, nullptr, nullptr, nullptr, nullptr, s, sl.partials, &np, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_leray(topt_ctx* c, const float* u, float* out, void* stream) {
  topt_status s0 = single_slab(c);
  if (s0 != TOPT_OK) return s0;
  if (!u || !out) return fail(TOPT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  launch_bchain(sl.g, u, sl.Z, c->p.alpha, c->p.reg_order, true, st);
  int np = 0;
  launch_assemble(sl.g, sl.Z, true, nullptr, nullptr, nullptr, nullptr, out, nullptr, sl.partials, &np, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_multidot(topt_ctx* c, const float* a, const float* const* bs, int32_t count, double* d_dots,
                          void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (emu(c)) return fail(TOPT_ERR_UNSUPPORTED, "multidot with emulated slabs");
  if (!a || !bs || !d_dots || count < 1 || count > kMaxVecs) return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  int np = 0;
  launch_multidot(a, bs, count, c->vecN, sl.partials, &np, st);
  launch_finalize_multi(sl.partials, 0, count, np, 1.0, d_dots, st);
  std::vector<double*> dd{d_dots};
  comm_allreduce(c, dd, count, false, st);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

topt_status topt_mix(topt_ctx* c, const float* q, const float* const* vs, const double* beta, int32_t count,
                     float* out, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (emu(c)) return fail(TOPT_ERR_UNSUPPORTED, "mix with emulated slabs");
  if (!q || !out || count < 0 || count > kMaxVecs || (count && (!vs || !beta)))
    return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  launch_mix(q, vs, beta, count, c->vecN, out, (cudaStream_t)stream);
  TOPT_CHECK_LAUNCH();
  return TOPT_OK;
}

// NGMRES(w) (Alg. 1) on the linear fixed-point map q(v) = v - omega g(v), g(v) = A v - b,
// A = I + alpha L (the v-chain, fp64) — the same Gram multi-dot, host LSQ and mixing kernels as
// topt_solve, on a problem whose NGMRES(infinity) iterates are GMRES's.
topt_status topt_linear_ngmres(topt_ctx* c, const float* b, double omega, float* v_inout, int32_t iters,
                               double* res, void* stream) {
  topt_status s0 = need_ws(c);
  if (s0 != TOPT_OK) return s0;
  if (c->comm.P > 1) return fail(TOPT_ERR_UNSUPPORTED, "linear NGMRES runs on one slab");
  if (c->p.model == TOPT_INCOMPRESSIBLE) return fail(TOPT_ERR_UNSUPPORTED, "A = I + alpha L needs a non-Leray model");
  if (!b || !v_inout || iters < 0 || !res) return fail(TOPT_ERR_INVALID_ARG, "bad argument");
  if (!aligned16(b) || !aligned16(v_inout)) return fail(TOPT_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  Slab& sl = c->slabs[0];
  const size_t V = c->vecN;
  const int W1 = c->p.window + 1;
  // g(x) = x + alpha L x - b into out
  auto apply_g = [&](const float* x, float* out) {
    std::vector<Io> io(1);
    io[0] = Io{nullptr, nullptr, x, nullptr, nullptr, nullptr, sl.pub(4), sl.intl(4)};
    run_vchain(c, io, st);
    launch_axpy(x, 1.0f, sl.utmp, V, out, st);
    launch_axpy(out, -1.0f, b, V, out, st);
  };
  auto norm2 = [&](const float* x, double& out) -> topt_status {
    std::vector<double> dd;
    topt_status rr = host_dots(c, [x](Slab&) { return x; }, {[x](Slab&) { return x; }}, dd, st);
    out = rr == TOPT_OK ? std::sqrt(dd[0]) : 0.0;
    return rr;
  };
  auto slotA = [&](int i) { return sl.hist + (size_t)(3 * i) * V; };
  auto slotB = [&](int i) { return sl.hist + (size_t)(3 * i + 1) * V; };
  std::deque<int> win;
  std::vector<std::vector<double>> H(W1, std::vector<double>(W1, 0.0));
  auto push = [&](const float* v, const float* g) -> topt_status {
    int slot;
    if ((int)win.size() < W1) slot = (int)win.size();
    else { slot = win.front(); win.pop_front(); }
    cudaMemcpyAsync(slotA(slot), v, V * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(slotB(slot), g, V * 4, cudaMemcpyDeviceToDevice, st);
    win.push_back(slot);
    std::vector<std::function<const float*(Slab&)>> bs;
    for (int s2 : win) bs.push_back([&, s2](Slab&) { return (const float*)slotB(s2); });
    std::vector<double> dd;
    topt_status rr = host_dots(c, [&, slot](Slab&) { return (const float*)slotB(slot); }, bs, dd, st);
    for (size_t i = 0; i < win.size() && rr == TOPT_OK; ++i) H[slot][win[i]] = H[win[i]][slot] = dd[i];
    return rr;
  };
  TOPT_CUDA(cudaMemcpyAsync(sl.vcur, v_inout, V * 4, cudaMemcpyDeviceToDevice, st));
  apply_g(sl.vcur, sl.gcur);
  topt_status r;
  if ((r = norm2(sl.gcur, res[0])) != TOPT_OK) return r;
  if ((r = push(sl.vcur, sl.gcur)) != TOPT_OK) return r;
  for (int k = 0; k < iters; ++k) {
    launch_axpy(sl.vcur, (float)(-omega), sl.gcur, V, sl.q, st);  // q = v - omega g
    apply_g(sl.q, sl.gq);
    const int m = (int)win.size();
    std::vector<std::function<const float*(Slab&)>> bs;
    for (int i = 0; i < m; ++i) { const int si = win[m - 1 - i]; bs.push_back([&, si](Slab&) { return (const float*)slotB(si); }); }
    bs.push_back([&](Slab&) { return (const float*)sl.gq; });
    std::vector<double> rd;
    if ((r = host_dots(c, [&](Slab&) { return (const float*)sl.gq; }, bs, rd, st)) != TOPT_OK) return r;
    const double gam = rd[m];
    std::vector<double> G(m * m), rhs(m);
    for (int i = 0; i < m; ++i) {
      rhs[i] = gam - rd[i];
      for (int j = 0; j < m; ++j) G[i * m + j] = gam - rd[i] - rd[j] + H[win[m - 1 - i]][win[m - 1 - j]];
    }
    std::vector<double> beta = lsq_from_gram(m, G, rhs);
    std::vector<const float*> vs;
    for (int i = 0; i < m; ++i) vs.push_back(slotA(win[m - 1 - i]));
    {
      Prof pr(c, K_MIX, (vs.size() + 2.0) * V * 4.0, 1, st);
      launch_mix(sl.q, vs.data(), beta.data(), m, V, sl.vnew, st);
    }
    apply_g(sl.vnew, sl.gnew);
    std::swap(sl.vcur, sl.vnew);
    std::swap(sl.gcur, sl.gnew);
    if ((r = norm2(sl.gcur, res[k + 1])) != TOPT_OK) return r;
    if ((r = push(sl.vcur, sl.gcur)) != TOPT_OK) return r;
  }
  TOPT_CUDA(cudaMemcpyAsync(v_inout, sl.vcur, V * 4, cudaMemcpyDeviceToDevice, st));
  TOPT_CUDA(cudaStreamSynchronize(st));
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

topt_status topt_set_graphs(topt_ctx* c, int32_t enable) {
  if (!c) return fail(TOPT_ERR_INVALID_ARG, "ctx is NULL");
  c->use_graphs = enable != 0;
  if (enable) c->slab_graphs_off = false;
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
// Every vector operation runs on every local slab; inner products are all-reduced.
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
  const double nF = ntot(c);
  const size_t nsl = c->slabs.size();
  std::memset(rep, 0, sizeof(*rep));
  const double t0 = now();
  double t_pde = 0.0, t_ls = 0.0, t_q = 0.0, t_f = 0.0;
  int grad_evals = 0, obj_evals = 0, nsteps = 0;
  std::deque<double> replay(c->replay.begin(), c->replay.end());
  topt_status r;
  using Acc = std::function<float*(Slab&)>;
  using CAcc = std::function<const float*(Slab&)>;

  // per-slab problem data (emulation: the user's whole-grid arrays are sliced)
  std::vector<const float*> m0s(nsl), m1s(nsl);
  for (size_t si = 0; si < nsl; ++si) {
    m0s[si] = emu(c) ? m0 + si * c->F : m0;
    m1s[si] = emu(c) ? m1 + si * c->F : m1;
  }
  auto io_at = [&](Acc v, Acc u, Acc g, Acc s, int set) {
    std::vector<Io> io(nsl);
    for (size_t si = 0; si < nsl; ++si) {
      Slab& sl = c->slabs[si];
      io[si] = Io{m0s[si], m1s[si], v(sl), u ? u(sl) : nullptr, g ? g(sl) : nullptr, s ? s(sl) : nullptr,
                  sl.pub(set), sl.intl(set)};
    }
    return io;
  };

  // history slot i: A = v (AA: r), B = g (AA: q), U = u (AA: u(q))
  auto slotA = [&](int i) { return Acc([i, V](Slab& s) { return s.hist + (size_t)(3 * i) * V; }); };
  auto slotB = [&](int i) { return Acc([i, V](Slab& s) { return s.hist + (size_t)(3 * i + 1) * V; }); };
  auto slotU = [&](int i) { return Acc([i, V](Slab& s) { return s.hist + (size_t)(3 * i + 2) * V; }); };
  auto cacc = [](Acc a) { return CAcc([a](Slab& s) { return (const float*)a(s); }); };
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
  auto copyv = [&](Acc dst, Acc src) {
    for (auto& sl : c->slabs) cudaMemcpyAsync(dst(sl), src(sl), V * 4, cudaMemcpyDeviceToDevice, st);
  };
  // push (a, b, u) and refresh the Gram row of b against the window
  auto push = [&](Acc a, Acc b, Acc u, bool gram) -> topt_status {
    const int slot = take_slot();
    copyv(slotA(slot), a);
    copyv(slotB(slot), b);
    copyv(slotU(slot), u);
    win.push_back(slot);
    if (!gram) return TOPT_OK;
    std::vector<CAcc> bs;
    for (int s2 : win) bs.push_back(cacc(slotB(s2)));
    std::vector<double> dd;
    topt_status rr = host_dots(c, cacc(slotB(slot)), bs, dd, st);
    if (rr != TOPT_OK) return rr;
    for (size_t i = 0; i < win.size(); ++i) H[slot][win[i]] = H[win[i]][slot] = dd[i];
    return TOPT_OK;
  };
  Acc Vc = [](Slab& s) { return s.vcur; }, Uc = [](Slab& s) { return s.ucur; };
  Acc Gc = [](Slab& s) { return s.gcur; }, Sc = [](Slab& s) { return s.scur; };
  Acc Q = [](Slab& s) { return s.q; }, Uq = [](Slab& s) { return s.uq; };
  Acc Gq = [](Slab& s) { return s.gq; }, Sq = [](Slab& s) { return s.sq; };
  Acc Vn = [](Slab& s) { return s.vnew; }, Un = [](Slab& s) { return s.unew; };
  Acc Gn = [](Slab& s) { return s.gnew; }, Sn = [](Slab& s) { return s.snew; };
  Acc Vt = [](Slab& s) { return s.vt; };

  // v^0, u^0 = alpha L v^0 (fp64 chain, once), g(v^0)
  if (emu(c)) stage_vec_in(c, v_inout, Vc, st);
  else TOPT_CUDA(cudaMemcpyAsync(c->slabs[0].vcur, v_inout, V * 4, cudaMemcpyDeviceToDevice, st));
  if (leray) leray_inplace(c, Vc, st);
  double te = now();
  {
    std::vector<Io> io = io_at(Vc, nullptr, Gc, Sc, 0);
    c->want_u = true;  // the old chain: u = alpha L v^0 is carried from here on
    forward_half(c, io, true, st);
    backward_half(c, io, st);  // computes u = alpha L v^0 into utmp
    c->want_u = false;
    for (auto& sl : c->slabs) cudaMemcpyAsync(sl.ucur, sl.utmp, V * 4, cudaMemcpyDeviceToDevice, st);
    TOPT_CHECK_LAUNCH();
  }
  ++grad_evals;
  HostScalars cur, qs, ns;
  if ((r = fetch(c, 0, cur, st)) != TOPT_OK) return r;
  t_pde += now() - te;
  const double g0 = cur.pub(TOPT_S_GRAD_INF);
  rep->grad_inf0 = g0;
  rep->dist0 = cur.pub(TOPT_S_DIST);
  if (!aa && (r = push(Vc, Gc, Uc, true)) != TOPT_OK) return r;

  // q-state helpers: v_q = v + rho s, u_q = u - rho (g - gbar)
  auto make_q = [&](double rho_) {
    float cst[3] = {0.f, 0.f, 0.f};
    for (int a = 0; a < c->d; ++a) cst[a] = (float)(rho_ * cur.in(I_SUMG + a) / nF);
    for (auto& sl : c->slabs) {
      launch_axpy(sl.vcur, (float)rho_, sl.scur, V, sl.q, st);
      launch_axpy_c(sl.ucur, (float)(-rho_), sl.gcur, V, c->d, cst, sl.uq, st);
    }
  };
  auto eval_into = [&](Acc v, Acc u, Acc g, Acc s, int set, HostScalars& out) -> topt_status {
    auto body = [&](cudaStream_t cs) -> topt_status { std::vector<Io> io = io_at(v, u, g, s, set);
                                                      return eval_gradient(c, io, cs); };
    Slab& s0 = c->slabs[0];
    const void* key[8] = {(const void*)3, m0s[0], m1s[0], v(s0), u ? u(s0) : nullptr, g(s0), s(s0),
                          (const void*)(intptr_t)set};
    topt_status rr = graphs_ok(c) ? graph_run(c, key, st, body) : body(st);
    if (rr != TOPT_OK) return rr;
    ++grad_evals;
    return fetch(c, set, out, st);
  };
  auto rotate = [&](float* Slab::*a, float* Slab::*b) {
    for (auto& sl : c->slabs) std::swap(sl.*a, sl.*b);
  };
  auto accept_q = [&]() {
    rotate(&Slab::vcur, &Slab::q);
    rotate(&Slab::ucur, &Slab::uq);
    rotate(&Slab::gcur, &Slab::gq);
    rotate(&Slab::scur, &Slab::sq);
    cur = qs;
  };
  auto eval_new = [&]() -> topt_status {
    if (leray) {
      leray_inplace(c, Vn, st);
      leray_inplace(c, Un, st);
    }
    topt_status rr = eval_into(Vn, Un, Gn, Sn, 3, ns);
    if (rr != TOPT_OK) return rr;
    rotate(&Slab::vcur, &Slab::vnew);
    rotate(&Slab::ucur, &Slab::unew);
    rotate(&Slab::gcur, &Slab::gnew);
    rotate(&Slab::scur, &Slab::snew);
    cur = ns;
    return TOPT_OK;
  };
  auto mix_into = [&](Acc out, Acc q, const std::vector<Acc>& vs, const std::vector<double>& beta) {
    for (auto& sl : c->slabs) {
      std::vector<const float*> p;
      for (auto& f : vs) p.push_back(f(sl));
      Prof pr(c, K_MIX, (p.size() + 2.0) * V * 4.0, 1, st);  // q and every v read, out written (a10)
      launch_mix(q(sl), p.data(), beta.data(), (int)p.size(), V, out(sl), st);
    }
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
        auto body = [&](cudaStream_t cs) -> topt_status { std::vector<Io> io = io_at(Q, nullptr, nullptr, nullptr, 1);
                                                          forward_half(c, io, false, cs);
                                                          TOPT_CHECK_LAUNCH();
                                                          return TOPT_OK; };
        const void* key[8] = {(const void*)4, m0s[0], m1s[0], Q(c->slabs[0]), nullptr, nullptr, nullptr, nullptr};
        if ((r = graphs_ok(c) ? graph_run(c, key, st, body) : body(st)) != TOPT_OK) return r;
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
    t_pde += now() - te;
    t_q += now() - te;
    if (!accepted) {
      exit_code = TOPT_STAGNATED;
      break;
    }

    const int period = P.sigma + P.tau;
    const bool fp_step = P.ordering == TOPT_ORDER_GA ? (k % period >= P.sigma) : (k % period < P.tau);
    const int wk = std::min(k, P.window);
    if (!aa) {
      te = now();
      if ((r = eval_into(Q, Uq, Gq, Sq, 2, qs)) != TOPT_OK) return r;  // g(q): both branches (R17)
      t_pde += now() - te;
      t_q += now() - te;
      if (fp_step) {
        accept_q();
      } else {
        // LSQ (Alg. 3 line 8): columns C_i = g_q - g(v^{k-i}), i = 0..w_k (R13), from the
        // fp64 Gram: G_ij = <g_q,g_q> - <g_q,g_i> - <g_q,g_j> + <g_i,g_j>, rhs_i = <C_i, g_q>
        const double tl = now();
        const int m = (int)win.size();  // == w_k + 1
        std::vector<CAcc> bs;
        for (int i = 0; i < m; ++i) bs.push_back(cacc(slotB(win[m - 1 - i])));  // i = 0 -> v^k
        bs.push_back(cacc(Gq));
        std::vector<double> rd;
        if ((r = host_dots(c, cacc(Gq), bs, rd, st)) != TOPT_OK) return r;
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
        std::vector<Acc> vs, us;
        for (int i = 0; i < m; ++i) {
          vs.push_back(slotA(win[m - 1 - i]));
          us.push_back(slotU(win[m - 1 - i]));
        }
        mix_into(Vn, Q, vs, beta);
        mix_into(Un, Uq, us, beta);
        te = now();
        if ((r = eval_new()) != TOPT_OK) return r;
        t_pde += now() - te;
        t_f += now() - te;
        ++nsteps;
      }
      (void)wk;
      if ((r = push(Vc, Gc, Uc, true)) != TOPT_OK) return r;
    } else {
      // AA (Alg. 2): r_k = v^k - q(v^k); LSQ over r_k - r_{k-i}, i = 1..w_k; mix q-images.
      // ONE multi-dot pass per step: <r_k, r_i> for every window slot and <r_k, r_k>; the
      // <r_i, r_j> come from the cached Gram H (rows filled when each r_i was pushed), exactly
      // the values a recomputation would give (fp64 sums of exact fp32 products, fixed order).
      for (auto& sl : c->slabs) launch_sub(sl.vcur, sl.q, V, sl.vt, st);  // r_k
      const int m = std::min((int)win.size(), wk);
      const int nw = (int)win.size();
      std::vector<double> rd;  // rd[i] = <r_k, r_{slot win[nw-1-i]}>, rd[nw] = <r_k, r_k>
      {
        const double tl = now();
        std::vector<CAcc> bs;
        for (int i = 0; i < nw; ++i) bs.push_back(cacc(slotA(win[nw - 1 - i])));
        bs.push_back(cacc(Vt));
        if ((r = host_dots(c, cacc(Vt), bs, rd, st)) != TOPT_OK) return r;
        t_ls += now() - tl;
      }
      const double gam = rd[nw];
      // push r_k (slot A), q (slot B), u(q) with its Gram row from rd
      auto push_r = [&]() {
        std::vector<int> old(win.begin(), win.end());
        const int slot = take_slot();
        copyv(slotA(slot), Vt);
        copyv(slotB(slot), Q);
        copyv(slotU(slot), Uq);
        for (int i = 0; i < nw; ++i) {
          const int so = old[nw - 1 - i];
          if (so == slot) continue;  // evicted
          H[slot][so] = H[so][slot] = rd[i];
        }
        H[slot][slot] = gam;
        win.push_back(slot);
      };
      if (!fp_step && m > 0) {
        const double tl = now();
        std::vector<double> G(m * m), rhs(m);
        for (int i = 0; i < m; ++i) {
          const int si = win[nw - 1 - i];
          rhs[i] = gam - rd[i];
          for (int j = 0; j < m; ++j) G[i * m + j] = gam - rd[i] - rd[j] + H[si][win[nw - 1 - j]];
        }
        std::vector<double> xi = lsq_from_gram(m, G, rhs);
        t_ls += now() - tl;
        std::vector<Acc> qv, qu;
        for (int i = 0; i < m; ++i) {
          qv.push_back(slotB(win[win.size() - 1 - i]));
          qu.push_back(slotU(win[win.size() - 1 - i]));
        }
        mix_into(Vn, Q, qv, xi);
        mix_into(Un, Uq, qu, xi);
        push_r();
        te = now();
        if ((r = eval_new()) != TOPT_OK) return r;
        t_pde += now() - te;
        t_f += now() - te;
        ++nsteps;
      } else {
        push_r();
        te = now();
        if ((r = eval_into(Q, Uq, Gq, Sq, 2, qs)) != TOPT_OK) return r;
        t_pde += now() - te;
        t_q += now() - te;
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
  if (emu(c)) stage_vec_out(c, cacc(Vc), v_inout, st);
  else TOPT_CUDA(cudaMemcpyAsync(v_inout, c->slabs[0].vcur, V * 4, cudaMemcpyDeviceToDevice, st));
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
  rep->t_q = t_q;
  rep->t_f = t_f;
  return TOPT_OK;
}

}  // extern "C"
