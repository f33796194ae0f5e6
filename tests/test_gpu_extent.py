"""Maximum extent per axis (include/topt.h: every extent a power of two up to 1024), through the C ABI
against the fp64 oracle.

Grids: the 2D config-1 recipe at 1024^2 (the displacement is ~4 cells there, so feet leave the
shared-memory halos and take the L1 gathers), and 3D boxes with one axis at 1024 — x (the
register-resident x-line FFTs at N = 1024, tiled SL kernels), y (strided lines at N = 1024) and z
(the last-axis passes incl. the merged pass at N = 1024; an 8-wide x axis takes the untiled SL
kernels).

Feet and forward sweeps are held to the bare per-operator tolerance.  Quantities that go through
fp32 spectral derivatives (the derivative itself, b, g, |g|_inf) may in addition carry twice the
error floor of an fp32 FFT at this extent ("fp32 FFT floor"): the rounding of a
length-N fp32 FFT leaves a white error of ~eps32 ||f|| per mode, which the derivative's symbol i k
(|k| up to N/2) lifts to ~eps32 N/(2 sqrt 3) ||f|| / ||df|| relative — 1.8e-5 for the 1024^2
config-1 phantom.  The floor is MEASURED here, independently of the CUDA path, by running the
oracle with its spectral derivative computed by torch's CPU complex64 FFT (no code shared with the
CUDA library); at the BASELINE configs' extents (<= 512) the bare 1e-5 holds and is what
tests/test_gpu_parity.py, test_gpu_fullsize.py and test_gpu_maxsize.py require."""
import numpy as np
import pytest
import torch

import test_gpu_parity as P
from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr
from oracle import spectral

pytestmark = pytest.mark.gpu
TOL = 1e-5

GRIDS = [
    (1, (1024, 1024)),      # 2D, largest extent on both axes
    (2, (1024, 8, 8)),      # x at 1024
    (3, (32, 1024, 8)),     # y at 1024
    (2, (8, 16, 1024)),     # z (last axis) at 1024, untiled SL path
]


def _deriv_fp32(grid, f, a):
    """The oracle's spectral derivative (symbol i k'_a, Nyquist zeroed: P:126, R3) with its FFTs in
    complex64 on the CPU (torch.fft): an fp32 FFT of our own choosing, sharing nothing with csrc/."""
    ax = np.ndim(f) - 1 - a
    n = np.shape(f)[ax]
    k = np.fft.fftfreq(n, d=1.0 / n)
    k[n // 2] = 0.0
    shape = [1] * np.ndim(f)
    shape[ax] = n
    F = torch.fft.fft(torch.tensor(np.asarray(f), dtype=torch.float32).to(torch.complex64), dim=ax)
    sym = torch.tensor((1j * k).reshape(shape), dtype=torch.complex64)
    return torch.fft.ifft(F * sym, dim=ax).real.double().numpy()


@pytest.mark.parametrize("cfg,n", GRIDS)
def test_feet_max_extent(cfg, n):
    P.test_feet(cfg, n)


@pytest.mark.parametrize("cfg,n", GRIDS)
@pytest.mark.parametrize("model", [0, 1])
def test_forward_max_extent(cfg, n, model):
    P.test_forward_trajectory(cfg, n, model)


@pytest.mark.parametrize("cfg,n", GRIDS)
def test_derivatives_max_extent(cfg, n):
    d = case(cfg, n)
    t = topt_for(d)
    f = d["m0"]
    for a in range(len(n)):
        out = host(t.derivative(dev(f), a))
        ref = spectral.deriv(d["grid"], f, a)
        floor = rel_l2(_deriv_fp32(d["grid"], f, a), ref)
        err = rel_l2(out, ref)
        print(cfg, n, a, f"err {err:.2e} fp32-FFT floor {floor:.2e}")
        assert err < TOL + 2.0 * floor, (a, err, floor)


def _fp32_floor(d, ref):
    """b, g and |g|_inf of the oracle's own trajectories (ref["m"], ref["lam"]) with the body force's
    gradients taken by the fp32 FFT (_deriv_fp32): the body-force formula (2.2) / R8 and g = alpha L v
    + b (P_L g for the incompressible model) as in oracle/gradient.py, only the derivative differs."""
    grid, nt, model = d["grid"], d["nt"], d["model"]
    w = ogr.trapezoid_weights(nt)
    grad32 = lambda f: np.stack([_deriv_fp32(grid, f, a) for a in range(grid.d)])
    b = np.zeros_like(ref["b"])
    for j in range(nt + 1):
        if model == 1:
            b -= w[j] * ref["m"][j] * grad32(ref["lam"][j])
        else:
            b += w[j] * ref["lam"][j] * grad32(ref["m"][j])
    g = d["alpha"] * spectral.apply_L(grid, d["v"], d["reg_order"]) + b
    if model == 2:
        g = spectral.leray(grid, g)
    return b, g, float(np.abs(g).max())


@pytest.mark.parametrize("cfg,n", GRIDS)
@pytest.mark.parametrize("model", [0, 1, 2])
def test_eval_gradient_max_extent(cfg, n, model):
    d = case(cfg, n, model=model)
    if model == 2:
        d["v"] = spectral.leray(d["grid"], d["v"]).astype(np.float32).astype(np.float64)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    lam, b = t.adjoint()
    lam, b, g, s = host(lam), host(b), host(g), host(s)
    nt = d["nt"]
    m = host(t.forward(dev(d["m0"]), dev(d["v"])))
    ref = ogr.evaluate(d["prob"], d["v"])
    b32, g32, ginf32 = _fp32_floor(d, ref)
    plam, pb, pg = P._propagated(d, ref, lam[nt])
    errs, allow = {}, {}
    for j in range(nt + 1):
        errs[f"m{j}"] = rel_l2(m[j], ref["m"][j])
        errs[f"lam{j}"] = rel_l2(lam[j], ref["lam"][j])
        allow[f"lam{j}"] = rel_l2(plam[j], ref["lam"][j])
    errs.update(b=rel_l2(b, ref["b"]), g=rel_l2(g, ref["g"]), s=rel_l2(s, ref["s"]))
    allow.update(b=rel_l2(pb, ref["b"]) + 2.0 * rel_l2(b32, ref["b"]),
                 g=rel_l2(pg, ref["g"]) + 2.0 * rel_l2(g32, ref["g"]))
    sd = t.scalars_dict(sc)
    for k in ("obj", "dist", "reg", "gs", "grad_inf"):
        errs[k] = abs(sd[k] - ref[k]) / (abs(ref[k]) + 1e-300)
    # |g|_inf: the same two terms in the max norm (the propagated forward error and the fp32 floor)
    allow["grad_inf"] = (abs(float(np.abs(pg).max()) - ref["grad_inf"]) + 2.0 * abs(ginf32 - ref["grad_inf"])) \
        / ref["grad_inf"]
    print(cfg, n, model, {k: f"{e:.2e}" + (f"/{allow[k]:.1e}" if allow.get(k) else "") for k, e in errs.items()})
    bad = {k: e for k, e in errs.items() if not e < TOL + allow.get(k, 0.0)}
    assert not bad, bad
