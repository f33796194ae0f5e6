/*
 * topt.h — C ABI of the B200-native GA-NGMRES transport-optimization hot path.
 *
 * Implements, on sm_100a, the hot path of arXiv 2510.08782: one
 * objective-plus-gradient evaluation per iteration (semi-Lagrangian forward
 * state solve, adjoint solve, body-force time integral, spectral
 * preconditioner (alpha L)^{-1}, Leray projection for the incompressible
 * model) together with the NGMRES window update (Gram inner products, host
 * fp64 least squares, mixing), driven by GA-NGMRES(w; sigma, tau) (Alg. 3).
 *
 * Citations: "P:n" = PAPER.md line n; "R<k>" = reading k in DESIGN.md §3.
 *
 * Conventions (every entry point)
 *  - Grid: Omega = [0, 2pi)^d, d in {2, 3}, n[i] cells along x_{i+1}, h_i = 2pi/n[i]
 *    (P:126-134).  Each n[i] must be a power of two in [8, 1024] (TOPT_ERR_UNSUPPORTED
 *    otherwise); for d == 2, n[2] must be 1.
 *  - Fields are fp32, C order [n[2]][n[1]][n[0]] (x fastest), DEVICE pointers unless
 *    an entry point's name ends in _host.  A vector field is d consecutive scalar
 *    fields (SoA): component c holds the x_{c+1} component.  "F" below = one scalar
 *    field = n[0]*n[1]*n[2] floats.  All pointers must be 16-byte aligned.
 *  - Reductions are accumulated in fp64 with a fixed order (bitwise reproducible).
 *  - Ownership: the caller owns every pointer passed in and the workspace.  The
 *    library never calls cudaMalloc: it owns only its context (host memory), a
 *    static device twiddle table, CUDA events and (world > 1) its NCCL communicator.
 *  - Streams: every device entry point enqueues on the caller's stream and returns
 *    without synchronising unless stated otherwise.
 *  - Errors: every call returns a topt_status; nothing throws across the ABI.
 *    topt_last_error() returns a thread-local message for the last failure.
 *    Non-convergence is not an error (reported in topt_report.exit).
 */
#ifndef TOPT_H_
#define TOPT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOPT_ABI_VERSION 1

typedef enum {
  TOPT_OK = 0,
  TOPT_ERR_INVALID_ARG = -1,  /* bad parameter / null pointer / misaligned pointer */
  TOPT_ERR_UNSUPPORTED = -2,  /* valid in the paper but not built (e.g. non power-of-two n) */
  TOPT_ERR_CUDA = -3,         /* a CUDA runtime error (message has the detail) */
  TOPT_ERR_NCCL = -4,         /* an NCCL error (world > 1) */
  TOPT_ERR_WORKSPACE = -5,    /* workspace missing or too small */
  TOPT_ERR_HALO = -6          /* internal: a foot left the sized z-slab window (never expected) */
} topt_status;

/* PDE constraint (P:35-41 advection; P:796-816 continuity; P:727-735 incompressible). */
typedef enum { TOPT_ADVECTION = 0, TOPT_CONTINUITY = 1, TOPT_INCOMPRESSIBLE = 2 } topt_model;

/* Exit state of a solve; ITER_CAP is the paper's "*". */
typedef enum { TOPT_CONVERGED = 0, TOPT_ITER_CAP = 1, TOPT_STAGNATED = 2 } topt_exit;

/* Acceleration: Alg. 3 GA-NGMRES or GA-AA (Alg. 2 under Alg. 3's schedule). */
typedef enum { TOPT_GA_NGMRES = 0, TOPT_GA_AA = 1 } topt_method;

/* Schedule ordering: Alg. 3 (FP when mod(k, sigma+tau) >= sigma) or the reverse
 * aNGMRES(w)[sigma]-FP[tau] (FP when mod(k, sigma+tau) < tau). */
typedef enum { TOPT_ORDER_GA = 0, TOPT_ORDER_REVERSE = 1 } topt_ordering;

typedef struct {
  int32_t dim;          /* d in {2, 3} */
  int32_t n[3];         /* cells per axis (x_1, x_2, x_3); n[2] = 1 when dim == 2 */
  int32_t nt;           /* number of time cells n_t >= 1 */
  int32_t model;        /* topt_model */
  int32_t reg_order;    /* p in {1, 2, 3}: L(k) = |k|^{2p} (R4; P:29 H2, P:734 H3) */
  double alpha;         /* regularisation weight alpha > 0 */
  int32_t window;       /* NGMRES depth w >= 0 */
  int32_t sigma;        /* NGMRES steps per period, >= 1 */
  int32_t tau;          /* FP steps per period, >= 0; (1, P-1) = "mixing period P" (R14) */
  int32_t method;       /* topt_method */
  int32_t ordering;     /* topt_ordering */
  int32_t max_iter;     /* n_iter (200) */
  double eps_rel;       /* relative l_inf gradient tolerance (5e-2) */
  double armijo_c;      /* Armijo constant c (1e-4) */
  int32_t max_backtracks; /* halvings before STAGNATED (R12: 50) */
} topt_params;

/* Solve report: the paper's table columns (P:354 caption) plus counters. */
typedef struct {
  double obj, dist, reg;      /* final objective and its parts */
  double grad_inf, grad_inf0; /* ||g(v^k)||_inf and ||g(v^0)||_inf */
  double rho;                 /* line-search memory at exit */
  int32_t iters;              /* completed updates (R16) */
  int32_t grad_evals;         /* objective+gradient evaluations */
  int32_t obj_evals;          /* forward-only objective evaluations (Armijo trials) */
  int32_t pde_solves;         /* 2 per gradient evaluation + 1 per trial */
  int32_t exit;               /* topt_exit */
  int32_t ngmres_steps;       /* accelerated steps taken */
  double t_total, t_pde, t_ls; /* seconds: time to solution, PDE evaluations, LSQ (host) */
  double t_q, t_f;              /* seconds: computing q(v^k) (Armijo trials + g(q)); evaluating
                                   the mixed iterate (the paper's q and f timer columns) */
  double dist0;                 /* dist at v^0 (the paper's "dist" column is dist / dist0) */
} topt_report;

typedef struct topt_ctx topt_ctx;

/* Scalar outputs of an evaluation, written as fp64 to a DEVICE array of
 * TOPT_NSCALARS doubles (index names below; topt_eval_gradient writes the reserved slots
 * 7..15 as zeros). */
#define TOPT_NSCALARS 16
enum {
  TOPT_S_OBJ = 0,      /* obj = dist + reg */
  TOPT_S_DIST = 1,     /* 1/2 <m^S - m1, m^S - m1>_h */
  TOPT_S_REG = 2,      /* alpha/2 <v, L v>_h (R23) */
  TOPT_S_GRAD_INF = 3, /* ||g||_inf over all d*n entries (R20) */
  TOPT_S_GS = 4,       /* <g, s>_h (Armijo slope) */
  TOPT_S_SLV = 5,      /* alpha <s, L v>_h   (linear term of reg(v + rho s)) */
  TOPT_S_SLS = 6       /* alpha <s, L s>_h   (quadratic term of reg(v + rho s)) */
};

/* ---- library / communicator --------------------------------------------------- */

/* ABI version (TOPT_ABI_VERSION). */
int32_t topt_abi_version(void);

/* Thread-local message describing the last failed call ("" if none). */
const char* topt_last_error(void);

/* Rank 0 only: a 128-byte NCCL unique id to broadcast (torch.distributed) before
 * topt_create on every rank.  Returns TOPT_ERR_UNSUPPORTED if built without NCCL. */
topt_status topt_get_unique_id(uint8_t id[128]);

/* Create a context for problem `p` on CUDA device `device`.  world >= 1 (a power of two)
 * splits the 3D grid into z-slabs of n[2]/world planes (BASELINE north_star):
 *  - id != NULL: NCCL mode, one slab per process (`rank`); fields passed to every call are
 *    this rank's slab [n[2]/world][n[1]][n[0]];
 *  - id == NULL, world > 1: all slabs emulated in this process on `device` (exchanges are
 *    device copies; rank must be 0); fields are whole-grid arrays.  Used to test that the
 *    decomposition reproduces world == 1.
 * Requires for world > 1: dim 3, n[1] and n[2] divisible by world, n[2]/world >= 4 (one
 * neighbour's 4 halo planes), n[0] >= 32, n[1] % 8 == 0.  Validates p
 * (TOPT_ERR_INVALID_ARG: odd/small n, alpha <= 0, sigma < 1, tau < 0, window < 0,
 * dim not in {2,3}, nt < 1, bad world).  Per-operator entry points (feet, forward,
 * get_adjoint, derivative, apply_precond, leray) need world == 1. */
topt_status topt_create(const topt_params* p, int32_t rank, int32_t world, const uint8_t* id,
                        int32_t device, topt_ctx** out);

/* Destroy a context (frees host state, events, communicator; not the workspace). */
topt_status topt_destroy(topt_ctx* ctx);

/* Bytes of device workspace the context needs (depends on n, nt, window, method). */
topt_status topt_workspace_size(const topt_ctx* ctx, size_t* bytes);

/* Bind a caller-allocated device workspace (>= topt_workspace_size bytes, 256-byte
 * aligned).  The workspace holds the trajectories, feet, FFT buffers and history. */
topt_status topt_bind_workspace(topt_ctx* ctx, void* dptr, size_t bytes);

/* Local z-slab of this rank: planes [z0, z0 + nz). */
topt_status topt_local_slab(const topt_ctx* ctx, int32_t* z0, int32_t* nz);

/* z-slabs (world > 1): transport of the z<->y all-to-all transposes.
 * COLLECTIVE with one process per GPU (every rank calls it, workspace bound; blocking): the
 * transport set is 1 only if every rank asked for 1 and holds the peer mappings, else 0 on
 * every rank — the ranks' collectives always match.
 * 0 (default) = pack + grouped ncclSend/ncclRecv + unpack; 1 = P2P pull: each rank reads its
 * chunks straight from the peers' slabs over NVLink (no pack / unpack passes), ordered by
 * one-byte all-reduce barriers.  With one process per GPU, transport 1 needs
 * topt_set_peer_workspaces first (topt_bind_workspace clears the mappings and resets 0); with emulated slabs (one process) it runs the same pull
 * kernel on the local slabs.  Transposes whose source is not in the workspace keep NCCL.
 * TOPT_ERR_INVALID_ARG for another value. */
topt_status topt_set_transport(topt_ctx* ctx, int32_t transport);

/* The transport in effect (0 or 1; -1 for a NULL context). */
int32_t topt_get_transport(const topt_ctx* ctx);

/* Peer workspaces for transport 1: bases[r] = rank r's bound workspace pointer (as passed to
 * its topt_bind_workspace) mapped into THIS process (CUDA IPC; bases[rank] = this rank's own),
 * count == world.  The pointers are borrowed: the caller keeps the mappings alive while the
 * context uses them.  count == 0 clears them.  TOPT_ERR_INVALID_ARG on a count mismatch. */
topt_status topt_set_peer_workspaces(topt_ctx* ctx, void* const* bases, int32_t count);

/* ---- solver --------------------------------------------------------------------- */

/* GA-NGMRES(w; sigma, tau) (Alg. 3) or GA-AA from v^0 = v_inout (the
 * paper uses v^0 = 0).  m0, m1: F each; v_inout: d*F, overwritten with the
 * final iterate.  Synchronous (host decisions: Armijo, LSQ); report filled on exit.
 * z-slabs (world > 1): every evaluation sizes its interpolation halo from the all-reduced
 * max |v_z| dt/h (trace) and max |delta_z| (SL steps): feet with |delta_z| < 3 cells read the
 * stored 4-plane halo, larger ones a window gathered from every slab they reach (up to a
 * whole period, then wrapped), so no trial is rejected for halo reasons (SL: no CFL cap).
 * TOPT_ERR_HALO would signal an internal error. */
topt_status topt_solve(topt_ctx* ctx, const float* m0, const float* m1, float* v_inout,
                       topt_report* report, void* stream);

/* Debug: force the Armijo step sequence of the next topt_solve (SURVEY §8(c)
 * "step replay").  count == 0 clears it.  rho is copied. */
topt_status topt_set_step_replay(topt_ctx* ctx, const double* rho, int32_t count);

/* ---- the benchmark unit ------------------------------------------------------------ */

/* One objective-plus-gradient evaluation at v: forward SL sweep, objective,
 * adjoint sweep, body force b = sum_j w_j lam^j grad m^j (continuity: -sum w_j pi^j
 * grad lam^j, R8), g = alpha L v + b (incompressible: P_L applied, R9) and
 * s = -(alpha L~)^{-1} g.  g, s: d*F device outputs; d_scalars: device
 * double[TOPT_NSCALARS].  Asynchronous. */
topt_status topt_eval_gradient(topt_ctx* ctx, const float* m0, const float* m1, const float* v,
                               float* g, float* s, double* d_scalars, void* stream);

/* Same evaluation from HOST buffers (pinned for best speed): copies m0, m1, v to the
 * workspace, evaluates, copies g back and the scalars to h_scalars (host double
 * [TOPT_NSCALARS]).  Synchronous (the end-to-end path timed by bench.py). */
topt_status topt_eval_gradient_host(topt_ctx* ctx, const float* m0_h, const float* m1_h,
                                    const float* v_h, float* g_h, double* h_scalars,
                                    void* stream);

/* Streaming form of topt_eval_gradient_host: ENQUEUES the copies of m0, m1, v, the
 * evaluation and the copies of g and the scalars back, and returns.  The library runs
 * them on its own copy-in, compute and copy-out streams with two device staging
 * buffers, so the transfers of consecutive calls overlap the evaluation of the call in
 * between; `stream` is made to wait for this call's results (the copy-in does not wait for
 * earlier work on `stream`: the inputs are host data).  The host buffers must stay valid
 * (inputs unmodified, outputs unread) until `stream` has been synchronised.
 * Single slab (world == 1) only: TOPT_ERR_UNSUPPORTED otherwise. */
topt_status topt_eval_gradient_host_async(topt_ctx* ctx, const float* m0_h, const float* m1_h,
                                          const float* v_h, float* g_h, double* h_scalars,
                                          void* stream);

/* Forward-only objective (what an Armijo trial costs): d_scalars[OBJ, DIST,
 * REG] written (REG by Parseval). Asynchronous. */
topt_status topt_objective(topt_ctx* ctx, const float* m0, const float* m1, const float* v,
                           double* d_scalars, void* stream);

/* Flow-map diagnostics (figure captions; reading R32): the
 * map y (foot at t = 0 of the characteristic ending at x at t = 1) as the composition of
 * the n_t backward semi-Lagrangian maps with the static RK2 foot, and det(grad y) by
 * spectral differentiation of the periodic displacement.  v: d*F device input;
 * y_disp: d*F device output, y(x) - x in radians; det: F device output.  Single slab
 * (world == 1) only: TOPT_ERR_UNSUPPORTED otherwise.  Asynchronous; uses the workspace
 * (do not overlap with an evaluation on another stream). */
topt_status topt_flow_map(topt_ctx* ctx, const float* v, float* y_disp, float* det, void* stream);

/* ---- operator entry points (per-operator parity) ----------------------------------- */

/* Characteristic feet as displacements in cells (R5, R6): delta_f = X - x (forward),
 * delta_a = Y - x (adjoint), d*F each. */
topt_status topt_feet(topt_ctx* ctx, const float* v, float* delta_f, float* delta_a, void* stream);

/* State trajectory: m_traj = [m^0, ..., m^{nt}] ((nt+1)*F) for velocity v (continuity:
 * with the Heun source factor, R7). */
topt_status topt_forward(topt_ctx* ctx, const float* m0, const float* v, float* m_traj,
                         void* stream);

/* After topt_eval_gradient: copy the adjoint trajectory [lam^0..lam^{nt}] ((nt+1)*F)
 * and the body force b (d*F) out of the workspace. Either pointer may be NULL. */
topt_status topt_get_adjoint(topt_ctx* ctx, float* lam_traj, float* body_force, void* stream);

/* out = d/dx_{axis+1} f (spectral, Nyquist zeroed, R3).  F each. */
topt_status topt_derivative(topt_ctx* ctx, const float* f, int32_t axis, float* out, void* stream);

/* s = -(alpha L~)^{-1} g (incompressible: with P_L), d*F each. */
topt_status topt_apply_precond(topt_ctx* ctx, const float* g, float* s, void* stream);

/* out = P_L u (Leray projector with the Nyquist-zeroed k', R3, R9), d*F each. */
topt_status topt_leray(topt_ctx* ctx, const float* u, float* out, void* stream);

/* ---- NGMRES kernels (used by topt_solve; exposed for parity) ------------------------ */

/* dots[i] = sum_x a(x) * b_i(x) over d*F entries, i = 0..count-1, fp64 (unweighted
 * l2, the LSQ norm of Alg. 1 line 5).  bs: host array of count device pointers. */
topt_status topt_multidot(topt_ctx* ctx, const float* a, const float* const* bs, int32_t count,
                          double* d_dots, void* stream);

/* out = (1 + sum beta_i) q - sum_i beta_i v_i over d*F entries (Alg. 1 line 6 /
 * Alg. 3 line 9).  vs: host array of count device pointers; beta: host doubles. */
topt_status topt_mix(topt_ctx* ctx, const float* q, const float* const* vs, const double* beta,
                     int32_t count, float* out, void* stream);

/* NGMRES(w) (Alg. 1) on the LINEAR fixed-point map q(v) = v - omega g(v),
 * g(v) = A v - b, A = I + alpha L (L of the context's reg_order, alpha L applied by the fp64
 * spectral chain, R4): the solver's Gram multi-dot, host fp64 LSQ and mixing kernels on a problem
 * whose NGMRES(infinity) iterates equal GMRES's.  b: d*F device input; v_inout: d*F
 * device, the start iterate in, v^{iters} out; res: HOST double[iters + 1], res[k] = ||g(v^k)||_2
 * (unweighted).  Single slab, advection or continuity context (TOPT_ERR_UNSUPPORTED otherwise).
 * Synchronous; uses the workspace. */
topt_status topt_linear_ngmres(topt_ctx* ctx, const float* b, double omega, float* v_inout, int32_t iters,
                               double* res, void* stream);

/* ---- instrumentation -------------------------------------------------------------------- */

/* enable != 0: bracket every launch group of the hot path with CUDA events on the caller's
 * stream (adds event records; use a separate, un-timed pass).  Clears accumulated stats.
 * Synchronizes the device. */
topt_status topt_profile(topt_ctx* ctx, int32_t enable);

/* enable != 0 (the default): topt_eval_gradient and topt_objective replay CUDA graphs keyed by
 * their pointer arguments (captured on first use; the workspace binding is baked in).  A single
 * slab captures the whole evaluation; with z-slabs (world > 1, NCCL or emulated) topt_eval_gradient
 * is captured in three segments between the host's two window decisions (max |v_z| before the trace, max |delta_z|
 * after it), each segment keyed by the decisions before it; the NCCL calls are
 * captured with the kernels (topt_objective runs eagerly on z-slabs).  enable == 0: every call runs eagerly (bitwise the same results).
 * Per-rank setting, but the ranks must agree (the collectives are the same either way).
 * Errors: TOPT_ERR_INVALID_ARG for a NULL ctx. */
topt_status topt_set_graphs(topt_ctx* ctx, int32_t enable);

/* Accumulated stats of kernel class `cls` (0..9; TOPT_ERR_INVALID_ARG past the end): class
 * name (static string), total event-timed ms, total ALGORITHMIC bytes (each operand read
 * once, each result written once per launch) and kernel launches.
 * Synchronizes on the recorded events. */
topt_status topt_kernel_stats(topt_ctx* ctx, int32_t cls, const char** name, double* ms, double* bytes,
                              int64_t* launches);

/* Number of kernels this library has launched since it was loaded (all contexts). */
int64_t topt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TOPT_H_ */
