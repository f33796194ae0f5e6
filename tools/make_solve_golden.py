"""Write tests/golden/solve_*.npz: fp64 ORACLE GA-NGMRES solves at the configs' native grids.

Calls only `oracle/` (the solver) and `synth/` (seeded inputs) — never the CUDA path.  Each case
is a 20-iteration solve from v^0 = 0 with eps = 0 (Alg. 3; north_star "after a fixed
20 iterations"), storing obj / dist / ||g||_inf, the accepted Armijo steps (for step replay,
SURVEY §8(c)), the relative-gradient history, the iteration count to the paper's stopping
tolerance eps = 5e-2 (a second, longer run when 20 iterations do not reach it) and
v encoded by tests/golden_io.py.  Inputs are rounded to fp32 once, exactly as
tests/gpu_common.case() hands them to both sides.

    python tools/make_solve_golden.py [--jobs 8] [--only c3_128_p1 ...]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")

EPS = 5e-2
N_COUNT = 60

# name -> (config recipe, grid, alpha override or None, w, sigma, tau)
CASES = {"c2_64": (2, (64, 64, 64), None, 5, 1, 0)}
for a in (1e-2, 1e-3, 1e-4):
    for w in (3, 5, 10):
        CASES[f"c4_64_a{a:.0e}_w{w}"] = (4, (64, 64, 64), a, w, 1, 0)
for p in (1, 2, 3, 4, 5):
    CASES[f"c3_128_p{p}"] = (3, (128, 128, 128), None, 5, 1, p - 1)
# config 5's recipe (advection, H2, alpha = 1e-3, n_t = 16, w = 10) at 64^3 (its 512^3 oracle solve
# would take days on the host)
CASES["c5_64"] = (5, (64, 64, 64), None, 10, 1, 0)
# config 4 at its native 256^3 (the benchmark's workload: continuity, H2, alpha = 1e-3, w = 5); hours of
# host time, run with all cores: NUMBA_NUM_THREADS=8 python tools/make_solve_golden.py --jobs 1 --only c4_256
CASES["c4_256"] = (4, (256, 256, 256), None, 5, 1, 0)


def run_case(name):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    from golden_io import encode_v
    from gpu_common import case
    from oracle import solver as osolver

    cfg, n, alpha, w, sigma, tau = CASES[name]
    d = case(cfg, n, alpha=alpha)
    t0 = time.time()
    r = osolver.solve(d["prob"], w=w, sigma=sigma, tau=tau, n_iter=20, eps_rel=0.0)
    conv = [k + 1 for k, g in enumerate(r.rel_grad) if g <= EPS]
    if conv:
        count, count_exit = conv[0], osolver.CONVERGED
    else:
        rc = osolver.solve(d["prob"], w=w, sigma=sigma, tau=tau, n_iter=N_COUNT, eps_rel=EPS)
        count, count_exit = rc.iters, rc.exit
    out = dict(config=cfg, n=np.array(n), alpha=float(d["alpha"]), w=w, sigma=sigma, tau=tau,
               iters=r.iters, exit=r.exit, obj=r.info["obj"], dist=r.info["dist"], reg=r.info["reg"],
               grad_inf=r.grad_inf, grad_inf0=r.grad_inf0, rel_grad=np.array(r.rel_grad),
               accepted=np.array(r.info["accepted"]), grad_evals=r.info["grad_evals"],
               obj_evals=r.info["obj_evals"], count=count, count_exit=count_exit, eps=EPS,
               oracle_seconds=time.time() - t0, **encode_v(r.v))
    np.savez_compressed(os.path.join(OUT, f"solve_{name}.npz"), **out)
    if os.environ.get("GOLDEN_RAW"):  # uncompressed copy of v for re-encoding (not committed)
        np.save(os.path.join(os.environ["GOLDEN_RAW"], f"v_{name}.npy"), r.v)
    return name, time.time() - t0, count, float(out["v_K"])


# fp32 resolution of the gradient: the GPU's body force carries a relative error up to
# ~1e-5 of ||b|| ~ ||g(v^0)||, so below a relative gradient of 1e-2 a step's direction is no longer
# determined to 1e-3 by an fp32 evaluation
RES32 = 1e-2


def kstar(name):
    """Store v at k* = the first iterate whose relative gradient is below RES32 (or the last one):
    the iterate the solve reaches with every step taken from a gradient above the fp32 resolution.
    The oracle solve is repeated for k* iterations (same path: deterministic)."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    from golden_io import encode_v
    from gpu_common import case
    from oracle import solver as osolver

    path = os.path.join(OUT, f"solve_{name}.npz")
    g = {k: v for k, v in np.load(path).items() if k not in ("sens", "sens_grad_noise")}
    rel = list(g["rel_grad"])
    ks = next((k + 1 for k, r in enumerate(rel) if r < RES32), len(rel))
    g["kstar"] = np.int64(ks)
    g["res32"] = np.float64(RES32)
    cfg, n, alpha, w, sigma, tau = CASES[name]
    d = case(cfg, n, alpha=alpha)
    t0 = time.time()
    if ks == int(g["iters"]):
        g.update({k.replace("v_", "vk_", 1): v for k, v in g.items() if k.startswith("v_")})
    else:
        r = osolver.solve(d["prob"], w=w, sigma=sigma, tau=tau, n_iter=ks, eps_rel=0.0)
        assert list(r.info["accepted"]) == list(g["accepted"][:ks])
        g["obj_kstar"] = np.float64(r.info["obj"])
        g.update(encode_v(r.v, prefix="vk"))
    g.setdefault("obj_kstar", g["obj"])
    np.savez_compressed(path, **g)
    return name, time.time() - t0, ks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--kstar", action="store_true", help="add k* and v(k*) to existing golden files")
    a = ap.parse_args()
    if a.kstar:
        names = a.only or sorted(CASES, key=lambda s: (-CASES[s][1][0], s))
        os.environ.setdefault("NUMBA_NUM_THREADS", "1")
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(min(a.jobs, len(names))) as pool:
            for name, sec, ks in pool.imap_unordered(kstar, names):
                print(f"{name}: k* = {ks} ({sec:.0f} s)", flush=True)
        return
    names = a.only or sorted(CASES, key=lambda s: (-CASES[s][1][0], s))  # largest grids first
    os.environ.setdefault("NUMBA_NUM_THREADS", "1")
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(min(a.jobs, len(names))) as pool:
        for name, sec, count, K in pool.imap_unordered(run_case, names):
            print(f"{name}: {sec:.0f} s, count {count}, K {K:.0f}", flush=True)


if __name__ == "__main__":
    main()
