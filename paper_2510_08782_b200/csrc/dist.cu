// dist.cu — z-slab communication: halo exchange, z<->y slab transposes, all-reduce.
//
// SURVEY §8(e) / BASELINE north_star: "halo exchange over NVLink sized from max|v|*dt for the
// interpolation, NCCL all-to-all transposes for the distributed FFT, and allreduce for the
// inner products".  Two transports behind one interface:
//   * NCCL (one slab per process, one process per GPU): grouped ncclSend/ncclRecv for halos
//     and the all-to-all, ncclAllReduce for scalars;
//   * emulation (all P slabs in one process on one GPU): the same data movement as device
//     copies — used by the tests to check that P slabs reproduce the single-slab result.
//   * P2P pull (transport 1, z<->y transposes): each rank reads its chunks straight from the
//     peers' slabs through CUDA-IPC-mapped workspaces (no pack / unpack passes, no NCCL
//     send/recv), ordered by one-byte all-reduce barriers before and after.
// Layouts: z-slab [nz/P][ny][nx] (halo'd inputs: [zh + nz/P + zh] planes); y-slab
// [nz][ny/P][nx].  The chunk exchanged between slabs r and q is nz/P x ny/P x nx elements.
#include <algorithm>
#include <cstdio>

#include "ctx.cuh"
#include "window.h"

namespace topt {

namespace {

#ifdef TOPT_WITH_NCCL
bool nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    fprintf(stderr, "topt: %s failed: %s\n", what, ncclGetErrorString(r));
    return false;
  }
  return true;
}
#endif

struct PtrList {
  double* p[64];
};

__global__ void k_allreduce_emul(PtrList L, int nslab, int count, int is_max) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double acc = L.p[0][i];
  for (int s = 1; s < nslab; ++s) acc = is_max ? fmax(acc, L.p[s][i]) : acc + L.p[s][i];
  for (int s = 0; s < nslab; ++s) L.p[s][i] = acc;
}

// P2P pull of one transpose (z->y if Z2Y, else y->z) for local rank r: 16-byte vectors of
// the P chunks, chunk q read from src[q] (rank q's buffer, local or peer-mapped).  z->y: my
// y-slab chunk q (planes of rank q, my rows) <- rank q's z-slab rows [r nyl, (r+1) nyl);
// y->z: my z-slab rows [q nyl, (q+1) nyl) <- rank q's y-slab chunk r.
struct SrcList {
  const char* p[64];
};
template <bool Z2Y>
__global__ void k_pull(char* __restrict__ dst, SrcList src, int P, int r, int nzl, int nyl, size_t rowb,
                       size_t pitch, size_t w, size_t chunk) {
  const size_t nv = rowb / 16, per = (size_t)nzl * nyl * nv, total = per * P;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / per);
    size_t j = i % per;
    const size_t v = j % nv;
    j /= nv;
    const int y = (int)(j % nyl), pl = (int)(j / nyl);
    size_t so, dof;
    if (Z2Y) {
      dof = q * chunk + pl * w + y * rowb + 16 * v;
      so = pl * pitch + ((size_t)r * nyl + y) * rowb + 16 * v;
    } else {
      so = r * chunk + pl * w + y * rowb + 16 * v;
      dof = pl * pitch + ((size_t)q * nyl + y) * rowb + 16 * v;
    }
    // .cv: peer memory is read around the local caches (no stale lines from an earlier pull)
    *reinterpret_cast<uint4*>(dst + dof) = __ldcv(reinterpret_cast<const uint4*>(src.p[q] + so));
  }
}

}  // namespace

// stream-ordered barrier over the ranks (every rank's earlier work on `st` is complete when
// it returns on the device): a one-byte all-reduce
static bool comm_barrier(topt_ctx* c, cudaStream_t st) {
#ifdef TOPT_WITH_NCCL
  char* b = c->slabs[0].sendbuf;
  return nccl_ok(ncclAllReduce(b, b, 1, ncclChar, ncclSum, c->comm.nccl, st), "ncclAllReduce(barrier)");
#else
  (void)c;
  (void)st;
  return false;
#endif
}

// a P2P pull needs the source inside the workspace (same offset on every rank); others (a
// caller's v, for instance) take the NCCL path
static bool pull_ok(const topt_ctx* c, const std::vector<const char*>& src) {
  if (c->comm.transport != 1) return false;
  if (c->comm.emulated()) return true;
  return (int)c->comm.peer_ws.size() == c->comm.P && src[0] >= c->ws && src[0] < c->ws + c->ws_bytes;
}

// z->y (Z2Y) or y->z transpose by P2P pull
static bool comm_pull(topt_ctx* c, bool z2y, const std::vector<const char*>& src, const std::vector<char*>& dst,
                      size_t eb, cudaStream_t st) {
  const Comm& cm = c->comm;
  const Slab& s0 = c->slabs[0];
  const int P = cm.P, nzl = s0.g.nz, nyl = s0.g.ny / P, nx = s0.g.nx;
  const size_t rowb = (size_t)nx * eb, w = nyl * rowb, pitch = (size_t)s0.g.ny * rowb, chunk = w * nzl;
  if (P > 64 || rowb % 16) return false;
  const bool emu = cm.emulated();
  if (!emu && !comm_barrier(c, st)) return false;  // every rank's source is complete
  const size_t vec = (size_t)P * nzl * nyl * (rowb / 16);
  const int blocks = (int)std::min<size_t>((vec + 255) / 256, 148 * 16);
  for (int r = 0; r < cm.nloc; ++r) {
    const int rank = emu ? r : c->slabs[0].index;
    SrcList L{};
    for (int q = 0; q < P; ++q)
      L.p[q] = emu ? src[q] : (q == rank ? src[0] : cm.peer_ws[q] + (src[0] - c->ws));
    if (z2y) k_pull<true><<<blocks, 256, 0, st>>>(dst[r], L, P, rank, nzl, nyl, rowb, pitch, w, chunk);
    else k_pull<false><<<blocks, 256, 0, st>>>(dst[r], L, P, rank, nzl, nyl, rowb, pitch, w, chunk);
    count_launch();
  }
  if (cudaGetLastError() != cudaSuccess) return false;
  return emu || comm_barrier(c, st);  // no rank overwrites a source another is still reading
}

// public helpers of the P2P transport for fused kernels (api.cu): is it usable, the rank-q
// image of a local workspace pointer, and the stream-ordered barrier (no-op when emulated)
bool comm_p2p_ready(const topt_ctx* c) {
  const Comm& cm = c->comm;
  return cm.transport == 1 && cm.P <= 8 && (cm.emulated() || (int)cm.peer_ws.size() == cm.P);
}
char* comm_peer(const topt_ctx* c, const void* p, int q) {
  const Comm& cm = c->comm;
  if (cm.emulated() || q == c->slabs[0].index) return (char*)p;
  return cm.peer_ws[q] + ((const char*)p - c->ws);
}
bool comm_fence(topt_ctx* c, cudaStream_t st) { return c->comm.emulated() || comm_barrier(c, st); }

// Halo planes of nf fields (field f of slab s at base[s] + f * fstride floats, layout
// [zh + nzl + zh] planes of `plane` floats): low halo <- previous slab's top zh local planes,
// high halo <- next slab's bottom zh local planes (ring, periodic in z).
bool comm_halo(topt_ctx* c, const std::vector<float*>& base, int nf, size_t fstride, cudaStream_t st) {
  const Comm& cm = c->comm;
  if (cm.P == 1) return true;
  const Slab& s0 = c->slabs[0];
  const int zh = s0.g.zh, nzl = s0.g.nz;
  const size_t pb = s0.plane * sizeof(float), hb = (size_t)zh * pb;
  if (cm.emulated()) {
    for (int f = 0; f < nf; ++f)
      for (int r = 0; r < cm.P; ++r) {
        const int prev = (r + cm.P - 1) % cm.P, next = (r + 1) % cm.P;
        float* B = base[r] + f * fstride;
        cudaMemcpyAsync(B, base[prev] + f * fstride + (size_t)nzl * s0.plane, hb, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(B + (size_t)(nzl + zh) * s0.plane, base[next] + f * fstride + (size_t)zh * s0.plane, hb,
                        cudaMemcpyDeviceToDevice, st);
      }
    return cudaGetLastError() == cudaSuccess;
  }
#ifdef TOPT_WITH_NCCL
  const int r = c->slabs[0].index, prev = (r + cm.P - 1) % cm.P, next = (r + 1) % cm.P;
  bool ok = nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (int f = 0; f < nf && ok; ++f) {
    float* B = base[0] + f * fstride;
    ok &= nccl_ok(ncclSend(B + (size_t)nzl * s0.plane, hb, ncclChar, next, cm.nccl, st), "ncclSend");
    ok &= nccl_ok(ncclRecv(B, hb, ncclChar, prev, cm.nccl, st), "ncclRecv");
    ok &= nccl_ok(ncclSend(B + (size_t)zh * s0.plane, hb, ncclChar, prev, cm.nccl, st), "ncclSend");
    ok &= nccl_ok(ncclRecv(B + (size_t)(nzl + zh) * s0.plane, hb, ncclChar, next, cm.nccl, st), "ncclRecv");
  }
  ok &= nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  return ok;
#else
  return false;
#endif
}

// Wide-halo window (multi-hop): slab r's window plane w (w < nzl + 2 zw) is global plane
// (z0_r - zw + w) mod nz, copied from the slab that owns it — up to every slab when zw > nzl.
// nf fields: field f of slab s at src[s] + f * fs floats (its LOCAL planes), written to slab s's
// win + f * (nzl + 2 zw) plane floats.  Runs of consecutive planes with one owner move as one
// copy (emulated) or one ncclSend / ncclRecv pair, issued in window order on both sides.

bool comm_window(topt_ctx* c, const std::vector<const float*>& src, size_t fs, int nf, int zw, cudaStream_t st) {
  const Comm& cm = c->comm;
  const Slab& s0 = c->slabs[0];
  const int nzl = s0.g.nz, nzg = nzl * cm.P;
  const size_t pl = s0.plane, ws = (size_t)(nzl + 2 * zw) * pl;
  if (zw > c->hcap) return false;
  if (cm.emulated()) {
    for (int r = 0; r < cm.P; ++r)
      for (const WindowRun& u : window_runs(r * nzl, nzl, nzg, zw))
        for (int f = 0; f < nf; ++f)
          cudaMemcpyAsync(c->slabs[r].win + f * ws + (size_t)u.w * pl, src[u.q] + f * fs + (size_t)u.lp * pl,
                          (size_t)u.len * pl * 4, cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError() == cudaSuccess;
  }
#ifdef TOPT_WITH_NCCL
  const int me = s0.index;
  float* win = c->slabs[0].win;
  for (const WindowRun& u : window_runs(me * nzl, nzl, nzg, zw))  // my own planes
    if (u.q == me)
      for (int f = 0; f < nf; ++f)
        cudaMemcpyAsync(win + f * ws + (size_t)u.w * pl, src[0] + f * fs + (size_t)u.lp * pl, (size_t)u.len * pl * 4,
                        cudaMemcpyDeviceToDevice, st);
  bool ok = nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (int r = 0; r < cm.P && ok; ++r) {
    if (r == me) continue;
    for (const WindowRun& u : window_runs(r * nzl, nzl, nzg, zw))  // what rank r needs from me
      if (u.q == me)
        for (int f = 0; f < nf; ++f)
          ok &= nccl_ok(ncclSend(src[0] + f * fs + (size_t)u.lp * pl, (size_t)u.len * pl * 4, ncclChar, r, cm.nccl, st),
                        "ncclSend");
  }
  for (const WindowRun& u : window_runs(me * nzl, nzl, nzg, zw))  // what I need from the others
    if (u.q != me)
      for (int f = 0; f < nf && ok; ++f)
        ok &= nccl_ok(ncclRecv(win + f * ws + (size_t)u.w * pl, (size_t)u.len * pl * 4, ncclChar, u.q, cm.nccl, st),
                      "ncclRecv");
  ok &= nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  return ok && cudaGetLastError() == cudaSuccess;
#else
  return false;
#endif
}

// z-slab -> y-slab transpose of one field per slab (element size eb bytes).
bool comm_z2y(topt_ctx* c, const std::vector<const char*>& src, const std::vector<char*>& dst, size_t eb,
              cudaStream_t st) {
  const Comm& cm = c->comm;
  if (pull_ok(c, src)) return comm_pull(c, true, src, dst, eb, st);
  const Slab& s0 = c->slabs[0];
  const int P = cm.P, nzl = s0.g.nz, nyl = s0.g.ny / P, nx = s0.g.nx;
  const size_t w = (size_t)nyl * nx * eb, spitch = (size_t)s0.g.ny * nx * eb, chunk = w * nzl;
  if (cm.emulated()) {
    for (int r = 0; r < P; ++r)
      for (int q = 0; q < P; ++q)
        cudaMemcpy2DAsync(dst[q] + r * chunk, w, src[r] + q * w, spitch, w, nzl, cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError() == cudaSuccess;
  }
#ifdef TOPT_WITH_NCCL
  char* sb = c->slabs[0].sendbuf;
  for (int q = 0; q < P; ++q)
    cudaMemcpy2DAsync(sb + q * chunk, w, src[0] + q * w, spitch, w, nzl, cudaMemcpyDeviceToDevice, st);
  bool ok = nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (int q = 0; q < P && ok; ++q) {
    ok &= nccl_ok(ncclSend(sb + q * chunk, chunk, ncclChar, q, cm.nccl, st), "ncclSend");
    ok &= nccl_ok(ncclRecv(dst[0] + q * chunk, chunk, ncclChar, q, cm.nccl, st), "ncclRecv");
  }
  ok &= nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  return ok;
#else
  return false;
#endif
}

// y-slab -> z-slab transpose of one field per slab.
bool comm_y2z(topt_ctx* c, const std::vector<const char*>& src, const std::vector<char*>& dst, size_t eb,
              cudaStream_t st) {
  const Comm& cm = c->comm;
  if (pull_ok(c, src)) return comm_pull(c, false, src, dst, eb, st);
  const Slab& s0 = c->slabs[0];
  const int P = cm.P, nzl = s0.g.nz, nyl = s0.g.ny / P, nx = s0.g.nx;
  const size_t w = (size_t)nyl * nx * eb, dpitch = (size_t)s0.g.ny * nx * eb, chunk = w * nzl;
  if (cm.emulated()) {
    for (int r = 0; r < P; ++r)
      for (int q = 0; q < P; ++q)
        cudaMemcpy2DAsync(dst[q] + r * w, dpitch, src[r] + q * chunk, w, w, nzl, cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError() == cudaSuccess;
  }
#ifdef TOPT_WITH_NCCL
  char* rb = c->slabs[0].sendbuf;
  bool ok = nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (int q = 0; q < P && ok; ++q) {
    ok &= nccl_ok(ncclSend(src[0] + q * chunk, chunk, ncclChar, q, cm.nccl, st), "ncclSend");
    ok &= nccl_ok(ncclRecv(rb + q * chunk, chunk, ncclChar, q, cm.nccl, st), "ncclRecv");
  }
  ok &= nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  for (int q = 0; q < P; ++q)
    cudaMemcpy2DAsync(dst[0] + q * w, dpitch, rb + q * chunk, w, w, nzl, cudaMemcpyDeviceToDevice, st);
  return ok;
#else
  return false;
#endif
}

// Collective agreement (one process per GPU): the minimum of `v` over the ranks, through the
// slab's scratch word (workspace bound), blocking.  Emulated / single slab: v itself.
int comm_agree_min(topt_ctx* c, int v) {
  const Comm& cm = c->comm;
  if (cm.P == 1 || cm.emulated()) return v;
#ifdef TOPT_WITH_NCCL
  int* d = reinterpret_cast<int*>(c->slabs[0].amax);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return 0;
  int out = 0;
  cudaMemcpyAsync(d, &v, sizeof(int), cudaMemcpyHostToDevice, st);
  const bool ok = nccl_ok(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, cm.nccl, st), "ncclAllReduce(agree)");
  cudaMemcpyAsync(&out, d, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return ok ? out : 0;
#else
  return 0;
#endif
}

// In-place all-reduce of `count` doubles at ptr[s] (per local slab).
bool comm_allreduce(topt_ctx* c, const std::vector<double*>& ptr, int count, bool is_max, cudaStream_t st) {
  const Comm& cm = c->comm;
  if (cm.P == 1 || count <= 0) return true;
  if (cm.emulated()) {
    PtrList L{};
    for (int s = 0; s < cm.P && s < 64; ++s) L.p[s] = ptr[s];
    k_allreduce_emul<<<1, 64, 0, st>>>(L, cm.P, count, is_max ? 1 : 0);
    count_launch();
    return cudaGetLastError() == cudaSuccess;
  }
#ifdef TOPT_WITH_NCCL
  return nccl_ok(ncclAllReduce(ptr[0], ptr[0], count, ncclDouble, is_max ? ncclMax : ncclSum, cm.nccl, st),
                 "ncclAllReduce");
#else
  return false;
#endif
}

}  // namespace topt
