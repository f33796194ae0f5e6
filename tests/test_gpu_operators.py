"""Per-operator parity on the small parity grids, each operator fed the GPU's OWN fp32 input to it
(rounded once, handed to the oracle in fp64), at the bare north_star tolerance 1e-5 — the same
structure as tests/test_gpu_fullsize.py at 256^3, for all three models:
  * lam^S = m1 - m^S (R1; continuity pi1 - pi^S, R8): bitwise (one correctly rounded fp32 subtraction);
  * every adjoint step lam^j = I[lam^{j+1}](Y) (* E_a for advection, R7; factor 1 otherwise, R8/R9);
  * the body force b = sum_j w_j lam^j grad m^j (continuity: -sum w_j pi^j grad lam^j, R8; R10);
  * g = alpha L v + b (incompressible: P_L(...), R9) and s = -(alpha L~)^{-1} g;
  * dist, reg, <g, s>_h and ||g||_inf from the GPU's fields.
Also the feet and every forward step (fed the GPU's m^j).  Whole fields, every time slice; the
configs' own grids for configs 2 (64^3, H1) and 3 (128^3, incompressible).  Cites: P:105-121 (gradient / adjoint), P:126 (trapezoid), P:136 (SL)."""
import numpy as np
import pytest
import torch

from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr
from oracle import spectral, transport
from oracle.interp import interp

pytestmark = pytest.mark.gpu
TOL = 1e-5

GRIDS = [
    (1, (64, 64)),
    (2, (32, 32, 32)),
    (2, (64, 16, 8)),
    (3, (32, 16, 64)),
    (4, (64, 64, 64)),
    (5, (16, 32, 64)),      # under-resolved (|k| <= 8 at the x Nyquist limit): per operator it is exact
]


def _run(cfg, n, model):
    d = case(cfg, n, model=model)
    if model == 2:
        d["v"] = spectral.leray(d["grid"], d["v"]).astype(np.float32).astype(np.float64)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    lam, b = t.adjoint()
    traj = t.forward(dev(d["m0"]), dev(d["v"]))
    df, da = t.feet(dev(d["v"]))
    torch.cuda.synchronize()
    return d, dict(g=host(g), s=host(s), sc=t.scalars_dict(sc), lam=host(lam), b=host(b), m=host(traj),
                   df=host(df), da=host(da))


CASES = [(c, n, m) for c, n in GRIDS for m in (0, 1, 2)]
CASES += [(2, (64, 64, 64), 0),      # config 2 at its native grid and model (H1)
          (3, (128, 128, 128), 2)]   # config 3 at its native grid and model (Leray, H2)


@pytest.mark.parametrize("cfg,n,model", CASES)
def test_operator_chain(cfg, n, model):
    d, r = _run(cfg, n, model)
    grid, nt, v = d["grid"], d["nt"], d["v"]
    lam, m = r["lam"], r["m"]
    # feet (R5, R6) and every forward step fed the GPU's m^j (continuity: Heun factor, R7)
    rf, ra = transport.feet(grid, v, nt)
    assert rel_l2(r["df"], rf) < TOL and rel_l2(r["da"], ra) < TOL, "feet"
    Ef = transport.source_factor_forward_continuity(grid, v, rf, nt) if model == 1 else 1.0
    assert np.array_equal(m[0], d["m0"])
    for j in range(nt):
        assert rel_l2(m[j + 1], interp(m[j], rf) * Ef) < TOL, ("forward step", j)
    # lam^S: fp32 subtraction of fp32 operands is the correctly rounded exact difference
    np.testing.assert_array_equal(lam[nt], (d["m1"] - m[nt]).astype(np.float32))
    # adjoint steps
    E = transport.source_factor_adjoint_advection(grid, v, ra, nt) if model == 0 else 1.0
    for j in range(nt - 1, -1, -1):
        ref = interp(lam[j + 1], ra) * E
        assert rel_l2(lam[j], ref) < TOL, ("adjoint step", j)
    # body force (trapezoid, R10)
    w = ogr.trapezoid_weights(nt)
    bref = np.zeros_like(r["b"])
    for j in range(nt + 1):
        if model == 1:
            bref -= w[j] * m[j] * spectral.grad(grid, lam[j])
        else:
            bref += w[j] * lam[j] * spectral.grad(grid, m[j])
    assert rel_l2(r["b"], bref) < TOL, "b"
    # gradient and preconditioned direction from the GPU's b and g
    gref = d["alpha"] * spectral.apply_L(grid, v, d["reg_order"]) + r["b"]
    if model == 2:
        gref = spectral.leray(grid, gref)
    assert rel_l2(r["g"], gref) < TOL, "g"
    sref = -spectral.apply_inv_alpha_L(grid, r["g"], d["alpha"], d["reg_order"])
    assert rel_l2(r["s"], sref) < TOL, "s"
    # scalars from the GPU's fields
    sc = r["sc"]
    res = m[nt] - d["m1"]
    dist = 0.5 * spectral.inner(grid, res, res)
    reg = spectral.reg_value(grid, v, d["alpha"], d["reg_order"])
    assert abs(sc["dist"] - dist) <= TOL * dist
    assert abs(sc["reg"] - reg) <= TOL * reg
    gs = spectral.inner(grid, r["g"], r["s"])
    assert abs(sc["gs"] - gs) <= TOL * abs(gs)
    assert abs(sc["grad_inf"] - np.max(np.abs(r["g"]))) <= TOL * sc["grad_inf"]
