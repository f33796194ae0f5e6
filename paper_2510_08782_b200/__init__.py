"""paper_2510_08782_b200 — B200-native GA-NGMRES for transport-constrained optimisation.

Thin Python binding of the C ABI in ``include/topt.h`` (libtopt.so, hand-written
sm_100a CUDA kernels).  PyTorch supplies device memory, streams and process
groups only; every step of the hot path runs in the library's kernels.  Names
follow PAPER.md (arXiv 2510.08782): m0, m1, v, alpha, nt, g, s, obj, GA-NGMRES
(w; sigma, tau).

Import fails loudly when the library is missing (no CPU fallback).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import LIB, Params, Report, ToptError, check

__all__ = ["Topt", "solve", "ToptError", "ADVECTION", "CONTINUITY", "INCOMPRESSIBLE", "SCALARS"]

ADVECTION, CONTINUITY, INCOMPRESSIBLE = 0, 1, 2
MODELS = {"advection": 0, "continuity": 1, "incompressible": 2}
SCALARS = {"obj": _lib.S_OBJ, "dist": _lib.S_DIST, "reg": _lib.S_REG, "grad_inf": _lib.S_GRAD_INF,
           "gs": _lib.S_GS, "slv": _lib.S_SLV, "sls": _lib.S_SLS}
EXIT = {0: "converged", 1: "iter_cap", 2: "stagnated"}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _f32(t, device, shape=None):
    t = torch.as_tensor(t)
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ToptError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not (t.is_cuda and t.device == torch.device(device) and t.dtype == torch.float32 and t.is_contiguous()):
        t = t.to(device=device, dtype=torch.float32).contiguous()
    return t


def _out(t, shape, dtype, device=None, pinned=False, name="output"):
    """Caller-supplied output buffer: the C ABI writes prod(shape) elements of `dtype` to it."""
    if not isinstance(t, torch.Tensor):
        raise ToptError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype or not t.is_contiguous() or t.numel() < int(torch.Size(shape).numel()):
        raise ToptError(f"{name}: need a contiguous {dtype} tensor of >= {tuple(shape)} elements, got "
                        f"{t.dtype} {tuple(t.shape)} contiguous={t.is_contiguous()}")
    if device is not None and t.device != torch.device(device):
        raise ToptError(f"{name} must live on {device}, not {t.device}")
    if pinned and (t.is_cuda or not t.is_pinned()):
        raise ToptError(f"{name} must be a pinned host tensor")
    return t


@dataclass
class Config:
    n: tuple               # paper order (n_1, ..., n_d)
    nt: int
    model: int = ADVECTION
    reg_order: int = 2
    alpha: float = 1e-2
    window: int = 5
    sigma: int = 1
    tau: int = 0
    method: int = 0        # 0 GA-NGMRES, 1 GA-AA
    ordering: int = 0      # 0 Alg. 3, 1 reverse (aNGMRES[sigma]-FP[tau])
    max_iter: int = 200
    eps_rel: float = 5e-2
    armijo_c: float = 1e-4
    max_backtracks: int = 50

    def params(self) -> Params:
        p = Params()
        d = len(self.n)
        p.dim = d
        nn = list(self.n) + [1] * (3 - d)
        for i in range(3):
            p.n[i] = int(nn[i])
        p.nt, p.model, p.reg_order, p.alpha = self.nt, self.model, self.reg_order, self.alpha
        p.window, p.sigma, p.tau = self.window, self.sigma, self.tau
        p.method, p.ordering, p.max_iter = self.method, self.ordering, self.max_iter
        p.eps_rel, p.armijo_c, p.max_backtracks = self.eps_rel, self.armijo_c, self.max_backtracks
        return p


class Topt:
    """One problem context bound to a CUDA device and a torch-allocated workspace.

    world > 1 splits the grid into z-slabs.  With ``unique_id`` (from
    ``get_unique_id`` on rank 0, broadcast with torch.distributed) each process owns one slab
    and exchanges over NCCL; fields passed in and out are that rank's slab
    [nz/world][ny][nx].  Without it, one process emulates all ``world`` slabs on one GPU
    (exchanges become device copies) and fields are whole-grid arrays — used to test that the
    decomposition reproduces the single-slab result."""

    def __init__(self, cfg: Config, device=None, rank: int = 0, world: int = 1, unique_id: bytes | None = None):
        if not torch.cuda.is_available():
            raise ToptError("a CUDA device is required (libtopt has no CPU path)")
        self.cfg = cfg
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.d = len(cfg.n)
        self.shape = tuple(reversed(cfg.n))
        self._p = cfg.params()
        ctx = ctypes.c_void_p()
        uid = ctypes.create_string_buffer(unique_id, 128) if unique_id else None
        with torch.cuda.device(self.device):
            check(LIB.topt_create(ctypes.byref(self._p), rank, world, uid, self.device.index,
                                  ctypes.byref(ctx)), "topt_create")
        self.ctx = ctx
        self.rank, self.world = rank, world
        z0, nz = ctypes.c_int32(), ctypes.c_int32()
        check(LIB.topt_local_slab(self.ctx, ctypes.byref(z0), ctypes.byref(nz)), "topt_local_slab")
        if self.d == 3:  # NCCL z-slabs: this rank's planes [z0, z0 + nz); emulation: the whole grid
            self.z0 = z0.value
            self.shape = (nz.value,) + self.shape[1:]
        else:
            self.z0 = 0
        nbytes = ctypes.c_size_t()
        check(LIB.topt_workspace_size(self.ctx, ctypes.byref(nbytes)), "topt_workspace_size")
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        off = (-base) % 256
        check(LIB.topt_bind_workspace(self.ctx, ctypes.c_void_p(base + off), nbytes.value),
              "topt_bind_workspace")
        self._ws_off = off
        self.scalars = torch.zeros(_lib.NSCALARS, dtype=torch.float64, device=self.device)

    # -- z-slab transport
    def set_transport(self, transport: str = "nccl"):
        """z<->y transposes: "nccl" (pack + send/recv + unpack) or "p2p" (pull from the peers'
        slabs; emulated slabs: the same pull kernel on the local slabs)."""
        check(LIB.topt_set_transport(self.ctx, {"nccl": 0, "p2p": 1}[transport]), "topt_set_transport")

    def enable_p2p(self, group=None):
        """One process per GPU: map every rank's workspace into this process (CUDA IPC through
        torch's CUDA tensor sharing, handles exchanged with torch.distributed) and switch the
        transposes to P2P pulls.  Collective: every rank calls it.  topt_set_transport agrees on the
        transport over the ranks, so when the mapping fails on any rank every rank stays on NCCL
        (this rank then re-raises the mapping error)."""
        err = None
        try:
            maps, offs = map_peer_tensors(self.workspace, self.rank, self.world, self._ws_off, group)
            self._peer_maps = maps  # keeps the mappings alive as long as this context
            bases = (ctypes.c_void_p * self.world)()
            for r in range(self.world):
                bases[r] = maps[r].data_ptr() + offs[r]
            check(LIB.topt_set_peer_workspaces(self.ctx, bases, self.world), "topt_set_peer_workspaces")
        except Exception as e:  # noqa: BLE001 — re-raised after the collective below
            err = e
        self.set_transport("p2p")  # collective; p2p only if every rank holds its mappings
        if err is not None:
            raise err

    @property
    def transport(self) -> str:
        return "p2p" if LIB.topt_get_transport(self.ctx) == 1 else "nccl"

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                LIB.topt_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # -- helpers
    def _vec(self):
        return torch.empty((self.d,) + self.shape, dtype=torch.float32, device=self.device)

    def _fld(self, k=1):
        return torch.empty(((k,) if k > 1 else ()) + self.shape, dtype=torch.float32, device=self.device)

    def scalars_dict(self, t=None):
        t = self.scalars if t is None else t
        h = t.cpu().tolist()
        return {k: h[i] for k, i in SCALARS.items()}

    # -- the benchmark unit
    def eval_gradient(self, m0, m1, v, g=None, s=None, scalars=None):
        m0, m1 = (_f32(x, self.device, self.shape) for x in (m0, m1))
        v = _f32(v, self.device, (self.d,) + self.shape)
        vshape = (self.d,) + self.shape
        g = self._vec() if g is None else _out(g, vshape, torch.float32, self.device, name="g")
        s = self._vec() if s is None else _out(s, vshape, torch.float32, self.device, name="s")
        sc = self.scalars if scalars is None else _out(scalars, (_lib.NSCALARS,), torch.float64, self.device,
                                                      name="scalars")
        check(LIB.topt_eval_gradient(self.ctx, _ptr(m0), _ptr(m1), _ptr(v), _ptr(g), _ptr(s), _ptr(sc),
                                     _stream()), "topt_eval_gradient")
        return g, s, sc

    def _host_args(self, m0_h, m1_h, v_h, g_h, scal_h):
        vshape = (self.d,) + self.shape
        for name, x, shp in (("m0", m0_h, self.shape), ("m1", m1_h, self.shape), ("v", v_h, vshape),
                             ("g", g_h, vshape)):
            _out(x, shp, torch.float32, pinned=True, name=name)
        _out(scal_h, (_lib.NSCALARS,), torch.float64, pinned=True, name="scalars")

    def eval_gradient_host(self, m0_h, m1_h, v_h, g_h, scal_h):
        """Host (pinned) buffers in, host buffers out; synchronous."""
        self._host_args(m0_h, m1_h, v_h, g_h, scal_h)
        check(LIB.topt_eval_gradient_host(self.ctx, _ptr(m0_h), _ptr(m1_h), _ptr(v_h), _ptr(g_h),
                                          _ptr(scal_h), _stream()), "topt_eval_gradient_host")

    def eval_gradient_host_async(self, m0_h, m1_h, v_h, g_h, scal_h):
        """Host (pinned) buffers; enqueues and returns (results valid after the current
        stream is synchronised).  Consecutive calls overlap transfers with evaluation."""
        self._host_args(m0_h, m1_h, v_h, g_h, scal_h)
        check(LIB.topt_eval_gradient_host_async(self.ctx, _ptr(m0_h), _ptr(m1_h), _ptr(v_h), _ptr(g_h),
                                                _ptr(scal_h), _stream()), "topt_eval_gradient_host_async")

    def objective(self, m0, m1, v):
        m0, m1, v = (_f32(x, self.device) for x in (m0, m1, v))
        sc = torch.zeros(_lib.NSCALARS, dtype=torch.float64, device=self.device)
        check(LIB.topt_objective(self.ctx, _ptr(m0), _ptr(m1), _ptr(v), _ptr(sc), _stream()), "topt_objective")
        return self.scalars_dict(sc)

    # -- diagnostics
    def flow_map(self, v):
        """(y - x in radians (d, *shape), det(grad y) (*shape)) — reading R32."""
        v = _f32(v, self.device)
        y, det = self._vec(), self._fld()
        check(LIB.topt_flow_map(self.ctx, _ptr(v), _ptr(y), _ptr(det), _stream()), "topt_flow_map")
        return y, det

    # -- operators
    def feet(self, v):
        v = _f32(v, self.device)
        df, da = self._vec(), self._vec()
        check(LIB.topt_feet(self.ctx, _ptr(v), _ptr(df), _ptr(da), _stream()), "topt_feet")
        return df, da

    def forward(self, m0, v):
        m0, v = _f32(m0, self.device), _f32(v, self.device)
        traj = self._fld(self.cfg.nt + 1)
        check(LIB.topt_forward(self.ctx, _ptr(m0), _ptr(v), _ptr(traj), _stream()), "topt_forward")
        return traj

    def adjoint(self):
        lam = self._fld(self.cfg.nt + 1)
        b = self._vec()
        check(LIB.topt_get_adjoint(self.ctx, _ptr(lam), _ptr(b), _stream()), "topt_get_adjoint")
        return lam, b

    def derivative(self, f, axis):
        f = _f32(f, self.device)
        out = self._fld()
        check(LIB.topt_derivative(self.ctx, _ptr(f), axis, _ptr(out), _stream()), "topt_derivative")
        return out

    def apply_precond(self, g):
        g = _f32(g, self.device)
        s = self._vec()
        check(LIB.topt_apply_precond(self.ctx, _ptr(g), _ptr(s), _stream()), "topt_apply_precond")
        return s

    def leray(self, u):
        u = _f32(u, self.device)
        out = self._vec()
        check(LIB.topt_leray(self.ctx, _ptr(u), _ptr(out), _stream()), "topt_leray")
        return out

    def multidot(self, a, bs):
        a = _f32(a, self.device)
        bs = [_f32(b, self.device) for b in bs]
        arr = (ctypes.c_void_p * len(bs))(*[b.data_ptr() for b in bs])
        out = torch.zeros(len(bs), dtype=torch.float64, device=self.device)
        check(LIB.topt_multidot(self.ctx, _ptr(a), arr, len(bs), _ptr(out), _stream()), "topt_multidot")
        return out

    def mix(self, q, vs, beta):
        q = _f32(q, self.device)
        vs = [_f32(x, self.device) for x in vs]
        arr = (ctypes.c_void_p * max(1, len(vs)))(*[x.data_ptr() for x in vs])
        b = (ctypes.c_double * max(1, len(beta)))(*[float(x) for x in beta])
        out = self._vec()
        check(LIB.topt_mix(self.ctx, _ptr(q), arr, b, len(vs), _ptr(out), _stream()), "topt_mix")
        return out

    def linear_ngmres(self, b, omega, iters, v0=None):
        """NGMRES(window) on q(v) = v - omega (A v - b), A = I + alpha L (topt_linear_ngmres).
        Returns (v, [||A v^k - b||_2 for k = 0..iters])."""
        vshape = (self.d,) + self.shape
        b = _f32(b, self.device, vshape)
        v = torch.zeros(vshape, dtype=torch.float32, device=self.device) if v0 is None \
            else _f32(v0, self.device, vshape).clone()
        res = (ctypes.c_double * (iters + 1))()
        check(LIB.topt_linear_ngmres(self.ctx, _ptr(b), float(omega), _ptr(v), int(iters), res, _stream()),
              "topt_linear_ngmres")
        return v, list(res)

    # -- instrumentation
    def profile(self, enable: bool = True):
        check(LIB.topt_profile(self.ctx, 1 if enable else 0), "topt_profile")

    def set_graphs(self, enable: bool = True):
        """CUDA-graph replay of evaluations (default on; z-slabs: segmented capture)."""
        check(LIB.topt_set_graphs(self.ctx, 1 if enable else 0), "topt_set_graphs")

    def kernel_stats(self):
        """Per kernel class: name, event-timed ms, algorithmic bytes, launches (since profile())."""
        out = []
        cls = 0
        while True:
            name = ctypes.c_char_p()
            ms, by, nl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
            st = LIB.topt_kernel_stats(self.ctx, cls, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(by),
                                       ctypes.byref(nl))
            if st != 0:
                break
            out.append({"name": name.value.decode(), "ms": ms.value, "bytes": by.value, "launches": nl.value})
            cls += 1
        return out

    @staticmethod
    def launch_count() -> int:
        return int(LIB.topt_launch_count())

    # -- solver
    def set_step_replay(self, rhos):
        arr = (ctypes.c_double * max(1, len(rhos)))(*[float(r) for r in rhos])
        check(LIB.topt_set_step_replay(self.ctx, arr, len(rhos)), "topt_set_step_replay")

    def solve(self, m0, m1, v0=None):
        m0, m1 = _f32(m0, self.device), _f32(m1, self.device)
        v = torch.zeros((self.d,) + self.shape, dtype=torch.float32, device=self.device) if v0 is None \
            else _f32(v0, self.device).clone()
        rep = Report()
        check(LIB.topt_solve(self.ctx, _ptr(m0), _ptr(m1), _ptr(v), ctypes.byref(rep), _stream()), "topt_solve")
        out = rep.as_dict()
        out["exit_name"] = EXIT.get(rep.exit, rep.exit)
        return v, out


def map_peer_tensors(t, rank: int, world: int, tag=None, group=None):
    """Collective over the process group: every rank's CUDA tensor `t` mapped into this process
    (CUDA IPC via torch's CUDA tensor sharing; rank `rank`'s own entry is `t` itself).  Returns
    (tensors, tags) indexed by rank; the mapped tensors must stay alive while they are used."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    objs = [None] * world
    dist.all_gather_object(objs, (reduce_tensor(t), tag), group=group)
    maps, tags = [], []
    for r, ((fn, args), tg) in enumerate(objs):
        maps.append(t if r == rank else fn(*args))
        tags.append(tg)
    return maps, tags


def get_unique_id() -> bytes:
    """NCCL unique id for topt_create (rank 0; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    check(LIB.topt_get_unique_id(buf), "topt_get_unique_id")
    return buf.raw


def solve(m0, m1, alpha, nt, model="advection", window=5, mixing_period=None, sigma=1, tau=0,
          reg_order=2, max_iter=200, eps_rel=5e-2, method="ngmres", ordering="ga", device=None):
    """GA-NGMRES(w; sigma, tau) from v^0 = 0 (Alg. 3).  ``mixing_period`` P maps to
    (sigma, tau) = (1, P - 1) (reading R14).  Returns (v, report)."""
    if mixing_period is not None:
        sigma, tau = 1, int(mixing_period) - 1
    m0t = torch.as_tensor(m0)
    n = tuple(reversed(m0t.shape))
    cfg = Config(n=n, nt=nt, model=MODELS.get(model, model), reg_order=reg_order, alpha=alpha,
                 window=window, sigma=sigma, tau=tau, method=0 if method == "ngmres" else 1,
                 ordering=0 if ordering == "ga" else 1, max_iter=max_iter, eps_rel=eps_rel)
    t = Topt(cfg, device=device)
    return t.solve(m0t, torch.as_tensor(m1))
