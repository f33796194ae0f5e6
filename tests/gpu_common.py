"""Shared helpers for the -m gpu parity tests: seeded inputs rounded to fp32 once, so the
oracle (fp64) and the CUDA path (fp32) see the SAME input values."""
import numpy as np
import torch

from oracle import gradient as ogr
from oracle.spectral import Grid
from synth import make_problem


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def case(config, n, scale=0.5, model=None, nt=None, alpha=None, reg_order=None):
    """Seeded problem of `config`'s recipe on grid n; inputs rounded to fp32.  Grids of 256^3 and up
    are generated on the GPU when one is present (the same closed forms, synth/phantoms.py)."""
    big = int(np.prod(n)) >= 256 ** 3 and torch.cuda.is_available()
    d = make_problem(config, n, device="cuda:0" if big else "cpu")
    if model is not None:
        d["model"] = model
    if nt is not None:
        d["nt"] = nt
    if alpha is not None:
        d["alpha"] = alpha
    if reg_order is not None:
        d["reg_order"] = reg_order
    d["m0"], d["m1"] = f32(d["m0"]), f32(d["m1"])
    d["v"] = f32(scale * d["vstar"])
    d["grid"] = Grid(tuple(d["n"]))
    d["prob"] = ogr.Problem(d["grid"], d["m0"], d["m1"], d["alpha"], d["nt"], d["model"], d["reg_order"])
    return d


def topt_for(d, world=1, **kw):
    import paper_2510_08782_b200 as topt
    cfg = topt.Config(n=tuple(d["n"]), nt=d["nt"], model=d["model"], reg_order=d["reg_order"],
                      alpha=d["alpha"], window=kw.pop("window", d.get("window", 5)),
                      sigma=kw.pop("sigma", d.get("sigma", 1)), tau=kw.pop("tau", d.get("tau", 0)), **kw)
    return topt.Topt(cfg, device="cuda:0", world=world)


def dev(x):
    return torch.tensor(np.asarray(x), dtype=torch.float32, device="cuda:0")


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()
