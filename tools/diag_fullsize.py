"""Diagnose high-|k| modes of g at 256^3 (config 4): u_GPU = g - b vs alpha L v (oracle, fp64)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_08782_b200 as topt
from oracle import spectral
from oracle.spectral import Grid
from synth import make_problem

d = make_problem(4, device="cuda:0")
n = tuple(d["n"]); grid = Grid(n)
f32 = lambda x: np.asarray(x, dtype=np.float32)
m0, m1, v = f32(d["m0"]), f32(d["m1"]), f32(d["vstar"])
t = topt.Topt(topt.Config(n=n, nt=d["nt"], model=d["model"], reg_order=d["reg_order"], alpha=d["alpha"]), device="cuda:0")
dev = lambda x: torch.tensor(x, device="cuda:0")
g, s, sc = t.eval_gradient(dev(m0), dev(m1), dev(v))
lam, b = t.adjoint()
torch.cuda.synchronize()
g = g.double().cpu().numpy(); b = b.double().cpu().numpy(); v = v.astype(np.float64)
print("rms g", np.sqrt(np.mean(g ** 2)), "rms b", np.sqrt(np.mean(b ** 2)))
for c in (1, 2):
    uref = d["alpha"] * np.real(np.fft.ifftn(spectral.reg_symbol(grid, 2) * np.fft.fftn(v[c])))
    ug = g[c] - b[c]
    print("comp", c, "rms uref", np.sqrt(np.mean(uref ** 2)), "rel L2 u", np.linalg.norm(ug - uref) / np.linalg.norm(uref))
    Uh, Rh = np.fft.fftn(ug), np.fft.fftn(uref)
    err = np.abs(Uh - Rh)
    print("  max mode err", err.max(), "at", np.unravel_index(err.argmax(), err.shape), "median", np.median(err))
    for k in [(128, 0, 0), (0, 128, 0), (0, 0, 128), (127, 0, 0), (100, 3, 5)]:
        idx = (k[2] % 256, k[1] % 256, k[0] % 256)
        print("  k", k, "|ref|", abs(Rh[idx]), "|err|", err[idx])
    # line structure of the error: x-Nyquist plane
    print("  err kx=128 plane max", err[:, :, 128].max(), "kx=127 plane max", err[:, :, 127].max(), "ky=128", err[:, 128, :].max(), "kz=128", err[128].max())
