"""Pins for oracle/gradient.py: closed forms at v = 0 and finite differences.

Paper passages: (1.1a) P:25-29, (2.2) P:105-108, adjoint (2.3) P:110-121 with
reading R1 (terminal sign), continuity P:796-816 with reading R8, incompressible
P:733-735 with reading R9, preconditioner P:168-175 / P:134.
"""
import numpy as np
import pytest

from oracle import gradient, spectral
from oracle.gradient import Problem
from oracle.spectral import Grid
from oracle.transport import ADVECTION, CONTINUITY, INCOMPRESSIBLE
from synth import make_problem


def _problem(n, nt, model, alpha=1e-2, p=2, cfg=1):
    d = make_problem(cfg, n)
    return Problem(Grid(tuple(n)), d["m0"], d["m1"], alpha, nt, model, p), d


def test_gradient_at_zero_closed_form_advection():
    """v = 0: m^j = m0, lam^j = m1 - m0, sum of trapezoid weights = 1 => g(0) = (m1 - m0) grad m0."""
    prob, _ = _problem((32, 32), 4, ADVECTION)
    r = gradient.evaluate(prob, np.zeros((2, 32, 32)))
    ref = (prob.m1 - prob.m0) * spectral.grad(prob.grid, prob.m0)
    np.testing.assert_allclose(r["g"], ref, atol=1e-15)
    assert r["reg"] == 0.0
    assert abs(r["dist"] - 0.5 * prob.grid.cell_volume * np.sum((prob.m1 - prob.m0) ** 2)) < 1e-15


def test_gradient_at_zero_closed_form_continuity_and_incompressible():
    prob, _ = _problem((32, 32), 4, CONTINUITY)
    r = gradient.evaluate(prob, np.zeros((2, 32, 32)))
    ref = -prob.m0 * spectral.grad(prob.grid, prob.m1 - prob.m0)
    np.testing.assert_allclose(r["g"], ref, atol=1e-15)
    prob, _ = _problem((32, 32), 4, INCOMPRESSIBLE)
    r = gradient.evaluate(prob, np.zeros((2, 32, 32)))
    ref = spectral.leray(prob.grid, (prob.m1 - prob.m0) * spectral.grad(prob.grid, prob.m0))
    np.testing.assert_allclose(r["g"], ref, atol=1e-14)
    assert np.max(np.abs(spectral.div(prob.grid, r["s"]))) < 1e-10


def test_search_direction_and_reg_term():
    """s = -(alpha L~)^{-1} g and <g, s>_h < 0 (descent); large alpha => g ~ alpha L v."""
    prob, d = _problem((32, 32), 4, ADVECTION)
    v = 0.5 * d["vstar"]
    r = gradient.evaluate(prob, v)
    back = -prob.alpha * spectral.apply_L(prob.grid, r["s"], 2)
    g0 = r["g"] - r["g"].mean(axis=(1, 2), keepdims=True)
    np.testing.assert_allclose(back, g0, atol=1e-10)
    assert r["gs"] < 0
    big = Problem(prob.grid, prob.m0, prob.m1, 1e4, 4, ADVECTION, 2)
    rb = gradient.evaluate(big, v)
    Lv = 1e4 * spectral.apply_L(prob.grid, v, 2)
    assert np.max(np.abs(rb["g"] - Lv)) < 1e-3 * np.max(np.abs(Lv))


def _fd_rel_error(n, nt, model, scale=0.5):
    prob, d = _problem(n, nt, model)
    g = prob.grid
    v = scale * d["vstar"]
    r = gradient.evaluate(prob, v)
    x1, x2 = g.coords()
    vt = np.stack([np.sin(x1 + 2 * x2 + 0.3) + 0.5 * np.cos(2 * x1), np.cos(x2 - x1 + 1.1)])
    if model == INCOMPRESSIBLE:
        vt = spectral.leray(g, vt)
    eps = 1e-4
    fp = gradient.objective(prob, v + eps * vt)["obj"]
    fm = gradient.objective(prob, v - eps * vt)["obj"]
    fd = (fp - fm) / (2 * eps)
    return abs(fd - spectral.inner(g, r["g"], vt)) / abs(fd)


@pytest.mark.parametrize("model", [ADVECTION, CONTINUITY, INCOMPRESSIBLE])
def test_gradient_matches_finite_differences(model):
    """Optimize-then-discretize: <g, v~> vs central FD agrees to the discretisation error
    (reading R22): <= 1e-2 at 64^2, and shrinking >= 2.5x per (2n, 2 n_t) refinement.
    A flipped terminal sign (the printed (2.3), R1) gives O(1) disagreement."""
    e64 = _fd_rel_error((64, 64), 4, model)
    e128 = _fd_rel_error((128, 128), 8, model)
    assert e64 < 1e-2
    assert e64 / e128 > 2.5


def test_printed_terminal_sign_fails_fd():
    """R1: with lam(1) = -(m1 - m(1)) literally, the gradient's data term flips sign."""
    prob, d = _problem((64, 64), 4, ADVECTION)
    v = 0.5 * d["vstar"]
    r = gradient.evaluate(prob, v)
    data = r["g"] - prob.alpha * spectral.apply_L(prob.grid, v, 2)
    flipped = prob.alpha * spectral.apply_L(prob.grid, v, 2) - data
    x1, x2 = prob.grid.coords()
    vt = np.stack([np.sin(x1 + 2 * x2 + 0.3), np.cos(x2 - x1 + 1.1)])
    eps = 1e-4
    fd = (gradient.objective(prob, v + eps * vt)["obj"] - gradient.objective(prob, v - eps * vt)["obj"]) / (2 * eps)
    good = abs(fd - spectral.inner(prob.grid, r["g"], vt)) / abs(fd)
    bad = abs(fd - spectral.inner(prob.grid, flipped, vt)) / abs(fd)
    assert good < 1e-2 and bad > 0.5


def _fd3(n, nt):
    prob, d = _problem((n, n, n), nt, ADVECTION, cfg=2)
    g = prob.grid
    v = 0.5 * d["vstar"]
    r = gradient.evaluate(prob, v)
    x1, x2, x3 = g.coords()
    vt = np.stack([np.sin(x1 + x3), np.cos(x2 - x1), np.sin(x3 + 2 * x2)])
    eps = 1e-4
    fd = (gradient.objective(prob, v + eps * vt)["obj"] - gradient.objective(prob, v - eps * vt)["obj"]) / (2 * eps)
    return abs(fd - spectral.inner(g, r["g"], vt)) / abs(fd)


def test_gradient_3d_fd():
    """3D (config-2 recipe): FD agreement improves >= 2.5x from 24^3/n_t=4 to 48^3/n_t=8."""
    e24, e48 = _fd3(24, 4), _fd3(48, 8)
    assert e48 < 2e-2 and e24 / e48 > 2.5
