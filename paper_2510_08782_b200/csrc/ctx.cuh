// ctx.cuh — library context: per-slab state and the z-slab communicator (not part of the ABI).
//
// z-slab decomposition (BASELINE north_star): the 3D grid is cut into P slabs of
// nz/P planes.  Each slab owns its fields; interpolated inputs carry zh = 4 halo planes per
// side (ring-periodic neighbour exchange before every SL step) — enough for feet with
// |delta_z| < 3 cells.  The halo is sized per evaluation from the all-reduced max |v_z| dt/h
// (trace) and max |delta_z| (SL steps): when a foot needs more, the step's input is gathered
// into a wider window (multi-hop: planes from every slab they live on, up to a whole period),
// so no foot is ever out of reach (SL has no CFL limit); z-derivatives and the z passes
// of the 3D FFTs run in a y-slab layout [nz][ny/P][nx] reached by an all-to-all transpose, and
// reductions are all-reduced.  One process may hold every slab (emulation on one GPU: the
// exchanges are device copies — used to test P-invariance) or exactly one (NCCL over NVLink).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.cuh"

#ifdef TOPT_WITH_NCCL
#include <nccl.h>
#endif

namespace topt {

constexpr int kSet = 32;  // doubles per scalar set: [0, 16) public, [16, 32) internal
constexpr int kSlabHalo = 4;

struct Slab {
  int index = 0;   // global slab index (rank)
  Geom g{};        // z-slab geometry (nz = local planes; zh = halo when P > 1)
  Geom gy{};       // y-slab geometry of the z passes (P > 1)
  size_t F = 0;    // local points
  size_t Fh = 0;   // local points incl. halo planes
  size_t plane = 0;
  float *m_traj{}, *lam_traj{}, *vh{}, *divv{};  // halo'd (Fh per slice / component)
  float *df{}, *da{}, *E{}, *b{}, *utmp{};
  float2* Z{};     // b-chain: 4 complex fields of F
  double2* Zv{};   // v-chain: 3 double-complex fields of F
  float2* Zy{};    // y-slab copies for P > 1
  double2* Zvy{};
  float* ytraj{};  // y-slab copies of the S+1 state and adjoint slices (P > 1)
  float* ytmp{};   // y-slab scratch (F)
  char* sendbuf{}; // NCCL transpose packing (16 F bytes)
  float *m0b{}, *m1b{}, *vb{}, *vt{};
  float *vcur{}, *gcur{}, *scur{}, *q{}, *gq{}, *sq{}, *vnew{}, *gnew{}, *snew{};
  float *ucur{}, *uq{}, *unew{};
  float* hist{};
  double* partials{};
  double* sc{};    // 5 sets of kSet
  double* dots{};
  int* haloerr{};
  unsigned* amax{};  // max |x| as float bits (window sizing)
  double* amaxd{};   // the same as a double (all-reduced)
  float* win{};      // wide-halo window: 3 fields of (nz + 2 hcap) planes
  double* pub(int set) const { return sc + set * kSet; }
  double* intl(int set) const { return sc + set * kSet + 16; }
};

// Communicator over the P slabs.  nloc == P: all slabs local (device copies); nloc == 1: NCCL.
// transport (z<->y transposes): 0 = pack + grouped ncclSend/ncclRecv + unpack; 1 = P2P pull —
// each rank reads its chunks straight from the peers' slabs (peer_ws: every rank's workspace
// base mapped into this process, CUDA IPC), stream-ordered by one-byte all-reduce barriers.
// Emulated slabs run the same pull kernel on the local slab pointers.
struct Comm {
  int P = 1;
  int nloc = 1;
  int transport = 0;
  std::vector<char*> peer_ws;
#ifdef TOPT_WITH_NCCL
  ncclComm_t nccl = nullptr;
#endif
  bool emulated() const { return nloc == P; }
};

}  // namespace topt

struct topt_ctx {
  topt_params p{};
  int rank = 0, world = 1, device = 0;
  int d = 3;
  int nzg = 1;
  double h[3]{}, dt = 0, cellvol = 0;
  std::vector<double> wts;
  size_t F = 0, vecN = 0;  // per slab
  char* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0, slab_bytes = 0;
  topt::Comm comm;
  std::vector<topt::Slab> slabs;
  std::vector<double> replay;
  // z-slab window sizing (P > 1): capacity hcap (covers a whole period), and the half-widths of
  // this evaluation's trace input (zw_v) and SL-step inputs (zw_m); 0 = the stored 4-plane halo
  int hcap = 0;
  int zw_v = 0, zw_m = 0;
  bool wrap_v = false, wrap_m = false;
  // side stream for work that depends on v only (eval_gradient, single slab)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_div = nullptr, ev_u = nullptr;
  bool div_pending = false, u_pending = false;
  bool vf_pending = false;  // side stream produces the fp64 forward v spectra (merged chain)
  bool want_u = false;      // the caller needs u = alpha L v in utmp (solver start): old chain
  // streaming host-buffer evaluations (topt_eval_gradient_host_async): two staging slots
  cudaStream_t h_in = nullptr, h_comp = nullptr, h_out = nullptr;
  cudaEvent_t ev_hfork = nullptr, ev_hin[2]{}, ev_hfree[2]{}, ev_hdone[2]{}, ev_hout[2]{};
  int hslot = 0;
  // CUDA graphs of topt_eval_gradient / topt_objective, keyed by their pointers (a captured
  // evaluation is replayed with one cudaGraphLaunch; the workspace binding is baked in)
  struct GraphEntry { const void* key[8]; cudaGraphExec_t exec; long long nlaunch; };
  std::vector<GraphEntry> graphs;
  cudaStream_t gcap = nullptr;  // capture stream (the caller's may be the legacy stream)
  cudaEvent_t ev_gcap = nullptr;
  bool use_graphs = true;
  // z-slab evaluations (P > 1) are captured in segments between the host's two window decisions
  // (max |v_z| before the trace, max |delta_z| after it): segment k is keyed by the user pointers
  // and the decisions 0..k-1; a replay launches segment k, reads decision k, picks segment k+1
  struct SegCap {
    bool on = false;            // capturing on gcap
    bool err = false;           // a capture failed: slab graphs are switched off, the evaluation re-run
    cudaStream_t user = nullptr;
    const void* base[6]{};
    std::vector<int> known;     // decisions already taken by this evaluation's replayed segments
    std::vector<int> dec;       // decisions taken in this capture
    long long l0 = 0;           // launch counter at the segment's start
  } segc;
  bool slab_graphs_off = false;
  // per-kernel-class timing (topt_profile / topt_kernel_stats)
  bool prof = false;
  struct Rec { int cls; cudaEvent_t a, b; double bytes; int launches; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double pms[16]{}, pbytes[16]{};
  long long plaunch[16]{};
};
