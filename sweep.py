"""Replica sweeps of GA-NGMRES / GA-AA on the synthetic 2D stand-in.

The paper's experiments are grids of solver settings on one registration problem:
  * wst   — w in {1, 5, 10, 15, 20, 25, 50} x (sigma, tau) in {(1,0), (5,1), (1,5), (5,5)}
            (tables T2/T3);
  * alpha — alpha in {1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4} x (sigma, tau) in {(5,1), (4,2)} x
            w in {10, 15, 20, 25};
  * mesh  — n in {64, 128, 256, 512} with n_t = 4, 8, 16, 32, alpha = 1e-3, w = 25,
            (sigma, tau) = (4, 2), eps_rel = 1e-3 (caption of the mesh table).
Every cell is an independent solve from v^0 = 0 (one replica per GPU: cells are dealt
round-robin to the ranks of `torchrun --nproc-per-node N sweep.py ...`, no collective on the
data path).  The problem is the config-1 recipe (BASELINE.json: 4 seeded Gaussians
transported by a divergence-free v*) — a stand-in for the paper's hands / nirep / rect data,
which are not available.  Each cell reports the paper's columns: #iter, #pdes, dist
(dist / dist(v^0)), grad (||g||_inf / ||g(v^0)||_inf), and the timers pdes (fraction of tts),
q, f, ls, tts ('*' when the iteration cap was hit).

    python sweep.py --grid wst --n 128 --max-iter 200 --eps 5e-2
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WST_W = [1, 5, 10, 15, 20, 25, 50]
WST_P = [(1, 0), (5, 1), (1, 5), (5, 5)]
ALPHA_A = [1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4]
ALPHA_P = [(5, 1), (4, 2)]
ALPHA_W = [10, 15, 20, 25]


def cells_for(grid: str, n: int, nt: int, alpha: float, w: int, sigma: int, tau: int):
    """The sweep's cells as dicts of Config overrides (paper order of the tables)."""
    if grid == "wst":
        return [dict(n=n, nt=nt, alpha=alpha, window=ww, sigma=s, tau=t) for (s, t) in WST_P for ww in WST_W]
    if grid == "alpha":
        return [dict(n=n, nt=nt, alpha=a, window=ww, sigma=s, tau=t)
                for a in ALPHA_A for (s, t) in ALPHA_P for ww in ALPHA_W]
    if grid == "mesh":
        return [dict(n=nn, nt=ss, alpha=1e-3, window=25, sigma=4, tau=2)
                for nn, ss in ((64, 4), (128, 8), (256, 16), (512, 32))]
    raise ValueError(grid)


def cells_of_rank(cells, rank: int, world: int):
    """Round-robin deal: cell i runs on rank i mod world (each cell exactly once)."""
    return [(i, c) for i, c in enumerate(cells) if i % world == rank]


def run_cell(cell, method: str, max_iter: int, eps: float, device):
    import numpy as np
    import torch

    import paper_2510_08782_b200 as topt
    from synth import make_problem

    d = make_problem(1, (cell["n"], cell["n"]), device=str(device))
    cfg = topt.Config(n=(cell["n"], cell["n"]), nt=cell["nt"], model=d["model"], reg_order=d["reg_order"],
                      alpha=cell["alpha"], window=cell["window"], sigma=cell["sigma"], tau=cell["tau"],
                      method=0 if method == "ngmres" else 1, max_iter=max_iter, eps_rel=eps)
    t = topt.Topt(cfg, device=device)
    m0 = torch.tensor(np.asarray(d["m0"], dtype=np.float32), device=device)
    m1 = torch.tensor(np.asarray(d["m1"], dtype=np.float32), device=device)
    _, rep = t.solve(m0, m1)
    del t
    tts = rep["t_total"]
    return {
        **cell, "method": method, "iters": rep["iters"], "pdes": rep["pde_solves"],
        "dist": rep["dist"] / rep["dist0"] if rep["dist0"] else 0.0,
        "grad": rep["grad_inf"] / rep["grad_inf0"] if rep["grad_inf0"] else 0.0,
        "t_pdes": rep["t_pde"], "pdes_frac": rep["t_pde"] / tts if tts else 0.0, "t_q": rep["t_q"],
        "t_f": rep["t_f"], "t_ls": rep["t_ls"], "tts": tts, "converged": rep["exit"] == 0, "exit": rep["exit_name"],
    }


def format_table(rows):
    head = f"{'run':>3} {'n':>4} {'nt':>3} {'alpha':>7} {'w':>3} {'(s,t)':>6} {'#iter':>5} {'#pdes':>6} " \
           f"{'dist':>10} {'grad':>10} {'pdes':>16} {'q':>8} {'f':>8} {'ls':>8} {'tts':>9}"
    out = [head]
    for i, r in enumerate(rows, 1):
        star = "" if r["converged"] else "*"
        out.append(f"{i:3d} {r['n']:4d} {r['nt']:3d} {r['alpha']:7.0e} {r['window']:3d} "
                   f"{'(%d,%d)' % (r['sigma'], r['tau']):>6} {r['iters']:5d} {r['pdes']:6d} {r['dist']:10.4e} "
                   f"{r['grad']:10.4e} {r['t_pdes']:8.3f} ({r['pdes_frac']:.2f}) {r['t_q']:8.3f} {r['t_f']:8.3f} "
                   f"{r['t_ls']:8.4f} {star + '%.3f' % r['tts']:>9}")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="wst", choices=["wst", "alpha", "mesh"])
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--nt", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=1e-2)
    ap.add_argument("--w", type=int, default=20)
    ap.add_argument("--sigma", type=int, default=5)
    ap.add_argument("--tau", type=int, default=1)
    ap.add_argument("--method", default="ngmres", choices=["ngmres", "aa"])
    ap.add_argument("--max-iter", type=int, default=200)
    ap.add_argument("--eps", type=float, default=5e-2)
    ap.add_argument("--json", default=None, help="write the rows as JSON lines here (rank 0)")
    args = ap.parse_args()

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    device = torch.device(f"cuda:{local}")
    torch.cuda.set_device(device)
    cells = cells_for(args.grid, args.n, args.nt, args.alpha, args.w, args.sigma, args.tau)
    mine = [(i, run_cell(c, args.method, args.max_iter, args.eps, device)) for i, c in cells_of_rank(cells, rank, world)]
    if world > 1:
        import torch.distributed as dist
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        mine = [x for part in allr for x in part]
        dist.destroy_process_group()
    if rank == 0:
        rows = [r for _, r in sorted(mine, key=lambda x: x[0])]
        print(format_table(rows), flush=True)
        if args.json:
            with open(args.json, "w") as f:
                for r in rows:
                    f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
