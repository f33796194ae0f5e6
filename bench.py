#!/usr/bin/env python
"""bench.py — gradient evaluations/s of the GA-NGMRES hot path on B200.

Metric (BASELINE.json): "gradient evals/s at 256^3 (fwd+adj+precond), % HBM roofline,
1/2/4/8 GPU".  Workload at N=1: BASELINE config 4 (256^3, continuity model, n_t = 8,
H2, alpha = 1e-3) — one step = one full objective-plus-gradient evaluation through the
C ABI (topt_eval_gradient: trace, forward SL sweep + objective, adjoint sweep, body
force, alpha L v and the preconditioner), inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl topt|reference]

N > 1 (torchrun): the 256^3 grid is split into N z-slabs, one per GPU, exchanging halos,
z<->y transposes and reductions over NCCL; value = evaluations of the one
problem / max-over-ranks device time (strong scaling).  --parallel replica instead runs one
independent replica per rank (weak scaling, no data-path collective).

--impl reference: the fp64 CPU oracle (oracle/, test infrastructure) timed on the host
cores on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gradient evals/s at 256^3 (fwd+adj+precond), % HBM roofline, 1/2/4/8 GPU"
UNIT = "evals/s"
CONFIG = 4


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _pass_model_bytes(cfg):
    """SURVEY §8(d) pass model, bytes per evaluation: d=3 A/C: (23 S + 53) F; I: (22 S + 38) F;
    d=2 A: (18 S + 38) F; F = 4 n bytes."""
    n = 1
    for x in cfg["n"]:
        n *= x
    F = 4.0 * n
    S = cfg["nt"]
    if len(cfg["n"]) == 2:
        return (18 * S + 38) * F
    if cfg["model"] == 2:
        return (22 * S + 38) * F
    return (23 * S + 53) * F


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        self.reader = threading.Thread(target=self._read, daemon=True)
        self.reader.start()
        t0 = time.time()  # the sampler is live before the timed region starts (short runs: >= 1 sample)
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)
        return self

    def _read(self):
        for l in self.proc.stdout:
            if l.strip():
                self.lines.append(l)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.reader.join(timeout=5)

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_init(backend="nccl"):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def share_unique_id(rank, world, make_id):
    """Rank 0 creates the 128-byte NCCL unique id; every rank receives it (torch.distributed)."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def slab_planes(nz, rank, world):
    """z-slab of `rank`: planes [z0, z0 + nz/world) (n[2] % world == 0)."""
    nzl = nz // world
    return rank * nzl, nzl


def slab_of(field, rank, world, vector=False):
    """This rank's z-slab of a whole-grid array (numpy [..., nz, ny, nx]), contiguous."""
    import numpy as np
    nz = field.shape[-3]
    z0, nzl = slab_planes(nz, rank, world)
    return np.ascontiguousarray(field[..., z0:z0 + nzl, :, :])


SLAB_CHECK_TOL = 1e-5  # north_star per-operator tolerance; emulated slabs agree to ~1e-7 (tests/test_gpu_slabs.py)
SLAB_CHECK_KEYS = ("dist", "reg", "gs", "grad_inf")


def slab_agreement(local, world, device=None, tol=SLAB_CHECK_TOL):
    """z-slab evaluation vs the single-GPU evaluation of the WHOLE grid (bench.py at N > 1, once, before
    timing).  `local` (per rank, from _slab_check): dl / rl = sums of squares of (g_slab - g_whole) and
    g_whole over this rank's planes, sc_slab / sc_full = the global scalars of both evaluations (dicts
    from Topt.scalars_dict), failed = 1.0 if this rank could not evaluate.  ONE all-reduce, the same
    on every rank whatever failed, so a rank's failure cannot desynchronise the collectives.  Returns
    the relative L2 of g over all slabs, the relative differences of dist, reg, <g,s>_h, ||g||_inf, ok."""
    vals = [float(local.get("dl", 0.0)), float(local.get("rl", 0.0)), float(local.get("failed", 1.0))]
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor(vals, dtype=torch.float64, device=device)
        dist.all_reduce(t)
        vals = t.tolist()
    dl, rl, failed = vals
    if failed > 0:
        return {"ok": False, "failed_ranks": int(round(failed)), **({"error": local["error"]} if "error" in local else {})}
    out = {"g_rel_l2": (dl / rl) ** 0.5 if rl > 0 else dl ** 0.5}
    for k in SLAB_CHECK_KEYS:  # global (all-reduced) scalars: the same on every rank
        a, b = local["sc_slab"][k], local["sc_full"][k]
        out[f"{k}_rel"] = abs(a - b) / max(abs(b), 1e-300)
    out.update(tol=tol, ok=bool(max(out.values()) <= tol))
    return out


def max_over_ranks(x, world, device=None):
    """Max of a float over ranks (device time of the slowest rank)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_eval_rate(n_sample, device):
    """One fp64 oracle evaluation of the config-4 recipe at n_sample^3: returns (seconds, scale)."""
    from oracle import gradient as ogr
    from oracle.spectral import Grid
    from synth import make_problem
    import numba
    numba.set_num_threads(_cpu_threads())
    # JIT warm-up at a tiny size (not timed)
    dw = make_problem(CONFIG, (16, 16, 16), device=device)
    ogr.evaluate(ogr.Problem(Grid((16, 16, 16)), dw["m0"], dw["m1"], dw["alpha"], dw["nt"], dw["model"],
                             dw["reg_order"]), dw["vstar"])
    d = make_problem(CONFIG, (n_sample,) * 3, device=device)
    prob = ogr.Problem(Grid((n_sample,) * 3), d["m0"], d["m1"], d["alpha"], d["nt"], d["model"], d["reg_order"])
    t0 = time.perf_counter()
    ogr.evaluate(prob, d["vstar"])
    return time.perf_counter() - t0, prob


def oracle_stage_sample(cfg_n, device):
    """The fp64 oracle (as it stands) timed at the FULL workload size on a bounded sample: one
    instance of every stage of its evaluation (oracle.gradient.evaluate), each weighted by
    how often one evaluation runs it (S = n_t): feet, the Heun factor (continuity), one forward and
    one adjoint SL step (x S each), one body-force slice (x S+1), the gradient and preconditioner.
    Returns (estimated seconds per evaluation, {stage: seconds})."""
    from oracle import gradient as ogr
    from oracle import spectral, transport
    from oracle.interp import interp
    from oracle.spectral import Grid
    from synth import make_problem
    import numba
    numba.set_num_threads(_cpu_threads())
    dw = make_problem(CONFIG, (16, 16, 16), device=device)  # JIT warm-up (not timed)
    ogr.evaluate(ogr.Problem(Grid((16, 16, 16)), dw["m0"], dw["m1"], dw["alpha"], dw["nt"], dw["model"],
                             dw["reg_order"]), dw["vstar"])
    d = make_problem(CONFIG, cfg_n, device=device)
    grid, S, v = Grid(tuple(d["n"])), d["nt"], d["vstar"]
    t = {}

    def clock(name, f):
        t0 = time.perf_counter()
        out = f()
        t[name] = time.perf_counter() - t0
        return out

    df, da = clock("feet", lambda: transport.feet(grid, v, S))
    E = clock("heun_factor", lambda: transport.source_factor_forward_continuity(grid, v, df, S))
    m1 = clock("forward_step", lambda: interp(d["m0"], df) * E)
    lam = clock("adjoint_step", lambda: interp(d["m1"] - m1, da))
    clock("body_force_slice", lambda: -m1 * spectral.grad(grid, lam))
    clock("gradient_precond", lambda: -spectral.apply_inv_alpha_L(
        grid, d["alpha"] * spectral.apply_L(grid, v, d["reg_order"]), d["alpha"], d["reg_order"]))
    count = {"feet": 1, "heun_factor": 1, "forward_step": S, "adjoint_step": S, "body_force_slice": S + 1,
             "gradient_precond": 1}
    return sum(t[k] * count[k] for k in t), t


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import torch
    from oracle import gradient as ogr
    from oracle.spectral import Grid
    from synth import make_problem
    import numba
    numba.set_num_threads(_cpu_threads())
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    # size the per-step sample so the whole run stays within ~3 minutes
    budget = 150.0
    steps = args.steps + args.warmup
    t_probe, _ = oracle_eval_rate(32, dev)
    per_point = t_probe / 32 ** 3
    n_s = 128
    while n_s > 32 and steps * per_point * n_s ** 3 * 1.3 > budget:
        n_s -= 16
    d = make_problem(CONFIG, (n_s,) * 3, device=dev)
    prob = ogr.Problem(Grid((n_s,) * 3), d["m0"], d["m1"], d["alpha"], d["nt"], d["model"], d["reg_order"])
    for _ in range(args.warmup):
        ogr.evaluate(prob, d["vstar"])
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ogr.evaluate(prob, d["vstar"])
        ts.append(time.perf_counter() - t0)
    scale = (n_s / 256.0) ** 3
    sec = sum(ts) / len(ts)
    value = scale / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
        "sample_ms_per_step": sec * 1e3,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config4_256^3_continuity_nt8_H2_alpha1e-3", "grid": [256, 256, 256]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle",
                         "sample": f"one fp64 oracle evaluation of the config-4 recipe at {n_s}^3 per step "
                                   f"(sample_ms_per_step); value EXTRAPOLATED by ({n_s}/256)^3 to the 256^3 "
                                   f"workload (ms_per_step = 1000 / value); bench.py's cpu_baseline times the "
                                   f"oracle's stages at 256^3 itself"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _slab_check(t, topt, d, cfgp, dev, rank, world, m0n, m1n, vn):
    """Evaluate once through the z-slab context t (eagerly, then twice through its segmented CUDA graphs,
    which must reproduce the eager result bitwise: graphs_diff) and once through a single-GPU context on
    the whole grid (every rank, its own GPU); local sums for slab_agreement (no collective here)."""
    import gc
    import torch
    f32 = lambda a: torch.tensor(a, dtype=torch.float32, device=dev)
    m0, m1, v = f32(m0n), f32(m1n), f32(vn)
    gs, ss, scs = torch.empty_like(v), torch.empty_like(v), torch.zeros(16, dtype=torch.float64, device=dev)
    t.set_graphs(False)  # the eager z-slab evaluation first ...
    t.eval_gradient(m0, m1, v, gs, ss, scs)
    sc_slab = t.scalars_dict(scs)
    ge, se, sce = gs.clone(), ss.clone(), scs.clone()
    t.set_graphs(True)  # ... then its segmented CUDA graphs, captured and replayed: bitwise the same
    same = True
    for _ in range(2):
        t.eval_gradient(m0, m1, v, gs, ss, scs)
        same = same and torch.equal(gs, ge) and torch.equal(ss, se) and torch.equal(scs, sce)
    full = topt.Topt(topt.Config(window=d["window"], **cfgp), device=dev)
    V = f32(d["vstar"])
    gf, sf, scf = full.eval_gradient(f32(d["m0"]), f32(d["m1"]), V)
    sc_full = full.scalars_dict(scf)
    z0, nzl = slab_planes(V.shape[-3], rank, world)
    gr = gf[..., z0:z0 + nzl, :, :].double()
    res = {"dl": float(((ge.double() - gr) ** 2).sum()), "rl": float((gr ** 2).sum()),
           "sc_slab": sc_slab, "sc_full": sc_full, "failed": 0.0, "graphs_diff": 0.0 if same else 1.0}
    del full, gf, sf, scf, V, gs, ss, gr, ge, se, sce
    gc.collect()
    torch.cuda.empty_cache()
    return res


def run_topt(args):
    import numpy as np
    import torch
    import paper_2510_08782_b200 as topt
    from synth import make_problem

    rank, world, local = _dist_init()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    n = tuple(args.n) if args.n else None
    d = make_problem(args.config, n, device=str(dev))
    torch.cuda.empty_cache()  # the generator's device temporaries (512^3: ~100 GB cached)
    cfgp = dict(n=tuple(d["n"]), nt=d["nt"], model=d["model"], reg_order=d["reg_order"], alpha=d["alpha"])
    slab = world > 1 and args.parallel == "slab"
    slab_error = None
    if slab:  # one z-slab per GPU over NCCL
        uid = share_unique_id(rank, world, topt.get_unique_id)
        t, err = None, 0.0
        try:
            t = topt.Topt(topt.Config(window=d["window"], **cfgp), device=dev, rank=rank, world=world,
                          unique_id=uid)
        except Exception as e:  # e.g. the NCCL communicator cannot be created on this node
            slab_error, err = f"{type(e).__name__}: {e}"[:200], 1.0
        if max_over_ranks(err, world, dev) > 0:  # every rank falls back together
            slab, t = False, None
            slab_error = slab_error or "z-slab context failed on another rank"
            if rank == 0:
                sys.stderr.write(f"bench: z-slab path unavailable ({slab_error}); running replicas\n")
    if slab and args.transport == "p2p":  # CUDA IPC mapping of the peers' workspaces
        try:
            t.enable_p2p()  # collective: every rank ends on the same transport
        except Exception as e:
            slab_error = f"p2p: {type(e).__name__}: {e}"[:200]
        if t.transport != "p2p":  # agreed over the ranks inside topt_set_transport
            args.transport = "nccl"
            slab_error = slab_error or "p2p mapping failed on another rank"
    zcheck = None
    if slab:
        m0n, m1n = slab_of(d["m0"], rank, world), slab_of(d["m1"], rank, world)
        vn = slab_of(d["vstar"], rank, world, vector=True)
        # once, before timing: this transport's z-slab evaluation against a single-GPU evaluation of
        # the whole grid on every rank (g over all slabs and the global scalars); a mismatch falls back
        # to replicas for the timed run and is recorded in the line
        try:
            local = _slab_check(t, topt, d, cfgp, dev, rank, world, m0n, m1n, vn)
        except Exception as e:
            local = {"failed": 1.0, "error": f"rank {rank}: {type(e).__name__}: {e}"[:200]}
        zcheck = slab_agreement(local, world, dev)
        if zcheck["ok"]:  # graph replay of the z-slab evaluation: on unless a rank saw it differ from eager
            gd = max_over_ranks(float(local.get("graphs_diff", 1.0)), world, dev)
            t.set_graphs(gd == 0.0)
            zcheck["graphs"] = "on" if gd == 0.0 else "off: replay differed from the eager evaluation"
        if not zcheck["ok"]:  # the same verdict on every rank (one all-reduce)
            slab, t = False, None
            slab_error = slab_error or f"z-slab check failed: {zcheck}"[:300]
            if rank == 0:
                sys.stderr.write(f"bench: {slab_error}; running replicas\n")
    if not slab:
        t = topt.Topt(topt.Config(window=d["window"], **cfgp), device=dev)
        m0n, m1n, vn = d["m0"], d["m1"], d["vstar"]
    m0 = torch.tensor(m0n, dtype=torch.float32, device=dev)
    m1 = torch.tensor(m1n, dtype=torch.float32, device=dev)
    v = torch.tensor(vn, dtype=torch.float32, device=dev)  # representative displacement
    g = torch.empty_like(v)
    s = torch.empty_like(v)
    sc = torch.zeros(16, dtype=torch.float64, device=dev)
    npts = int(np.prod(m0n.shape))  # points of this rank
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            t.eval_gradient(m0, m1, v, g, s, sc)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = topt.Topt.launch_count()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        e0, e1 = ev[0], ev[-1]
        e0.record(stream)
        for k in range(args.steps):  # one event per step boundary (no synchronisation inside)
            t.eval_gradient(m0, m1, v, g, s, sc)
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        launches = topt.Topt.launch_count() - l0
        ms = e0.elapsed_time(e1)
        step_ms = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps))
    ms = max_over_ranks(ms, world, dev)
    ms_per_step = ms / args.steps
    evals = args.steps if slab else world * args.steps  # slab: the ranks share one problem
    value = evals / (ms / 1e3)

    # per-kernel-class breakdown, separate (un-timed) pass with event brackets
    t.profile(True)
    for _ in range(args.steps):
        t.eval_gradient(m0, m1, v, g, s, sc)
    stats = t.kernel_stats()
    t.profile(False)
    peak, peak_kind = _peaks()
    kern = [x for x in stats if x["ms"] > 0]
    total_ms = sum(x["ms"] for x in kern)
    dom = max((x for x in kern if x["bytes"] > 0), key=lambda x: x["ms"])
    achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            ent = tr.get("classes", {}).get(dom["name"])
            if ent and ent.get("grid") == list(d["n"]):
                traffic = ent.get("bytes_per_launch")
        except Exception:
            traffic = None
    per_launch_bytes = dom["bytes"] / max(1, dom["launches"])
    # The SL kernels are bound by shared-memory bandwidth, not HBM: a tricubic
    # point reads 64 taps x 4 B from shared memory.  Peak = 148 SMs x 128 B/clk x the SM clock
    # measured during the timed region (B300_MICROARCH.md: 128/N B/cyc/SM crossbar).
    smem_roofline = None
    sl = next((x for x in kern if x["name"] == "sl_step"), None)
    if sl and sl["ms"] > 0:
        taps_bytes = 64 * 4.0 * npts * sl["launches"]
        sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        speak = nsm * 128.0 * sm_mhz * 1e6 / 1e9
        sach = taps_bytes / (sl["ms"] / 1e3) / 1e9
        smem_roofline = {"kernel": "sl_step", "bound": "smem", "achieved": round(sach, 1), "peak": round(speak, 1),
                         "unit": "GB/s", "frac": round(sach / speak, 4),
                         "bytes_per_point": 256, "peak_kind": f"derived: {nsm} SMs x 128 B/clk x {sm_mhz:.0f} MHz"}
    roofline = {"bound": "hbm", "kernel": dom["name"], "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": per_launch_bytes, "peak_kind": peak_kind,
                "share_of_step": round(dom["ms"] / total_ms, 4) if total_ms else None}
    profile_ms_per_step = total_ms / args.steps  # kernels serialised (no side-stream overlap)
    breakdown = {x["name"]: {"share": round(x["ms"] / total_ms, 4),
                             "GB/s": round(x["bytes"] / (x["ms"] / 1e3) / 1e9, 1) if x["bytes"] else None,
                             "launches_per_step": x["launches"] / args.steps} for x in kern}
    model_bytes = _pass_model_bytes(cfgp) / (world if slab else 1)  # per rank

    # end to end through the public API with HOST buffers (pinned): H2D m0, m1, v; D2H g + scalars,
    # streamed (topt_eval_gradient_host_async: step k's copies overlap step k+-1's evaluation)
    e2e = None
    if not args.no_e2e:
        m0h = torch.tensor(m0n, dtype=torch.float32).pin_memory()
        m1h = torch.tensor(m1n, dtype=torch.float32).pin_memory()
        vh = torch.tensor(vn, dtype=torch.float32).pin_memory()
        gh = torch.empty_like(vh).pin_memory()
        sch = torch.zeros(16, dtype=torch.float64).pin_memory()
        # one slab: the streaming call (transfers of step k+-1 overlap step k); z-slabs over NCCL:
        # the synchronous call (the library's copy streams are single-slab)
        host_eval = t.eval_gradient_host if slab else t.eval_gradient_host_async
        for _ in range(max(1, args.warmup)):
            host_eval(m0h, m1h, vh, gh, sch)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):  # every step: H2D m0, m1, v; evaluate; D2H g + scalars
            host_eval(m0h, m1h, vh, gh, sch)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(f0.elapsed_time(f1), world, dev)
        e2e = {"value": evals / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(4 * npts * (2 + len(d["n"]))),
               "d2h_bytes_per_step": int(4 * npts * len(d["n"]) + 16 * 8)}
        # context for e2e (outside the timed region): this box's pinned-copy bandwidth for the same
        # buffers, H2D of the step's inputs and D2H of g (plain torch copies), and the evaluations/s
        # that the slower direction alone would allow
        try:
            bufs = [torch.empty_like(x, device=dev) for x in (m0h, m1h, vh)]
            gd = torch.empty_like(vh, device=dev)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c2 = torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                c0.record(stream)
                for b_, h_ in zip(bufs, (m0h, m1h, vh)):
                    b_.copy_(h_, non_blocking=True)
                c1.record(stream)
                gh.copy_(gd, non_blocking=True)
                c2.record(stream)
                torch.cuda.synchronize()
            h2d_s, d2h_s = c0.elapsed_time(c1) / 1e3, c1.elapsed_time(c2) / 1e3
            # both directions at once, as in the streamed steady state (full-duplex PCIe; the host side
            # may not sustain both at full rate)
            so = torch.cuda.Stream(device=dev)
            for _ in range(2):
                so.wait_stream(stream)
                c0.record(stream)
                with torch.cuda.stream(so):
                    gh.copy_(gd, non_blocking=True)
                for b_, h_ in zip(bufs, (m0h, m1h, vh)):
                    b_.copy_(h_, non_blocking=True)
                stream.wait_stream(so)
                c1.record(stream)
                torch.cuda.synchronize()
            dup_s = c0.elapsed_time(c1) / 1e3
            e2e["pcie"] = {"h2d_GB/s": round(e2e["h2d_bytes_per_step"] / h2d_s / 1e9, 1),
                           "d2h_GB/s": round(4 * npts * len(d["n"]) / d2h_s / 1e9, 1),
                           "duplex_ms": round(dup_s * 1e3, 3),
                           "copy_bound_evals/s_per_rank": round(1.0 / max(h2d_s, d2h_s, dup_s), 1)}
            del bufs, gd
        except Exception as e:  # context only: never fails the line
            e2e["pcie"] = {"error": f"{type(e).__name__}"}

    # GA-NGMRES iterations (Armijo trials, Gram inner products, host LSQ,
    # mixing, stop test) on the same problem from v^0 = 0, after freeing the evaluation context
    solver = None
    if args.solver_iters > 0:
        host_eval = None  # a bound method keeps the evaluation context (and its workspace) alive
        del t
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        kw = dict(window=d["window"], sigma=d.get("sigma", 1), tau=d.get("tau", 0), max_iter=args.solver_iters,
                  eps_rel=0.0, **cfgp)
        if slab:  # a fresh NCCL unique id per communicator
            uid2 = share_unique_id(rank, world, topt.get_unique_id)
            ts = topt.Topt(topt.Config(**kw), device=dev, rank=rank, world=world, unique_id=uid2)
            if args.transport == "p2p":  # collective; falls back to NCCL on every rank together
                try:
                    ts.enable_p2p()
                except Exception:
                    pass
        else:
            ts = topt.Topt(topt.Config(**kw), device=dev)
        ts.solve(m0, m1)  # warm-up
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = ts.solve(m0, m1)
        torch.cuda.synchronize()
        sec = max_over_ranks(time.perf_counter() - t0, world, dev)
        ts.profile(True)
        ts.solve(m0, m1)
        st = {x["name"]: x for x in ts.kernel_stats()}
        ts.profile(False)
        gbs = lambda k: round(st[k]["bytes"] / (st[k]["ms"] / 1e3) / 1e9, 1) if st.get(k, {}).get("ms") else None
        F = npts * 4.0
        solver = {"method": f"GA-NGMRES(w={kw['window']}; sigma={kw['sigma']}, tau={kw['tau']})",
                  "iterations": rep["iters"], "wall_s": round(sec, 4),
                  "ms_per_iteration": round(1e3 * sec / max(1, rep["iters"]), 3),
                  "iterations_per_s": round(rep["iters"] / sec, 3),
                  "grad_evals": rep["grad_evals"], "obj_evals": rep["obj_evals"],
                  "ls_share": round(rep["t_ls"] / rep["t_total"], 4) if rep["t_total"] else None,
                  "gram_GB/s": gbs("ngmres_gram"), "mix_GB/s": gbs("ngmres_mix"),
                  "ngmres_step_bytes_model": (3 * (kw["window"] + 2) + 4) * len(d["n"]) * F}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sec, stages = oracle_stage_sample(tuple(cfgp["n"]), str(dev))
        cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle",
               "sample": f"fp64 oracle (oracle/, numba + numpy, as it stands) on the {'x'.join(map(str, cfgp['n']))} "
                         f"config-{args.config} workload itself: one instance of each evaluation stage timed, "
                         f"weighted by its count per evaluation (S = {cfgp['nt']}): "
                         + ", ".join(f"{k} {v:.2f} s" for k, v in stages.items()),
               "sec_per_eval_estimated": round(sec, 3)}

    if rank == 0:
        wl = {1: "config1_2D_64^2_advection_nt4_H2", 2: "config2_64^3_advection_nt4_H1",
              3: "config3_128^3_incompressible_nt8_H2", 4: "config4_256^3_continuity_nt8_H2_alpha1e-3",
              5: "config5_512^3_advection_nt16_H2"}[args.config]
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "step_ms": {"median": round(statistics.median(step_ms), 4),
                        "p10": round(step_ms[int(0.1 * (len(step_ms) - 1))], 4),
                        "p90": round(step_ms[int(round(0.9 * (len(step_ms) - 1)))], 4),
                        "rank0_only": world > 1},
            "scaling": "strong" if slab else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl, "grid": list(d["n"]), "nt": d["nt"], "model": d["model"],
                       "reg_order": d["reg_order"], "alpha": d["alpha"],
                       "parallelism": (f"zslab{world}" if slab else f"replicas{world}") if world > 1 else "single",
                       **({"transport": args.transport} if slab else {}),
                       **({"zslab_error": slab_error} if slab_error else {}),
                       **({"zslab_check": zcheck} if zcheck is not None else {}),
                       "l2": "inputs larger than L2 (~15 GB of HBM traffic per evaluation vs 126 MB L2)"},
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roofline,
            "smem_roofline": smem_roofline,
            "cpu_baseline": cpu,
            "hbm_frac_pass_model": round(model_bytes * (value if slab else value / world) / (peak * 1e9), 4),
            "pass_model_bytes_per_eval": model_bytes,
            "kernels": breakdown,
            "profile_ms_per_step_serialised": round(profile_ms_per_step, 4),
            "solver": solver,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="topt", choices=["topt", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--n", type=int, nargs="*", default=None, help="override grid (paper order)")
    ap.add_argument("--cpu-n", type=int, default=128, help="oracle sample grid for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--solver-iters", type=int, default=4, help="GA-NGMRES iterations timed (0: skip)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="z-slabs: z<->y transposes by NCCL send/recv or by P2P pulls over CUDA IPC")
    ap.add_argument("--parallel", default="slab", choices=["slab", "replica"],
                    help="N > 1: z-slabs over NCCL (one problem) or independent replicas")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_topt(args)


if __name__ == "__main__":
    main()
