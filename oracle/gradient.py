"""Objective, reduced gradient and preconditioned direction (fp64).  TEST INFRASTRUCTURE ONLY.

PAPER.md anchors:
  (1.1a) obj(v) = 1/2 ||m(1) - m1||^2_{L2} + alpha/2 ||Delta v||^2
  (2.2)  g(v)   = alpha Delta^2 v + int_0^1 lam grad m dt
  (2.3)  adjoint final-value problem
  (2.5)/(2.6) s = -(alpha L)^{-1} g  (RPGD direction)
  trapezoidal rule in time; kernel of L fixed to 1
  continuity model (3.1); incompressible: div v = 0

Readings:
  R1  terminal adjoint lam(1) = m1 - m(1) (the printed -(m1 - m) flips the data
      term; derived from the Lagrangian)
  R4  L(k) = |k|^{2p}, p = reg_order (H1/H2/H3)
  R8  continuity: lam(1) = pi1 - pi(1), b = - int pi grad lam dt
  R9  incompressible: g = P_L(alpha L v + b), s = -(alpha L~)^{-1} g (in range(P_L))
  R10 trapezoid weights dt/2 at the end points, dt inside
  R11 discrete norms: h^d-weighted sums; ||g||_inf over all d*n entries (R20)
  R23 reg value = alpha/2 <v, L v>_h (Parseval)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import spectral, transport
from .spectral import Grid
from .transport import ADVECTION, CONTINUITY, INCOMPRESSIBLE


@dataclass
class Problem:
    grid: Grid
    m0: np.ndarray
    m1: np.ndarray
    alpha: float
    nt: int
    model: int = ADVECTION
    reg_order: int = 2

    def __post_init__(self):
        self.m0 = np.asarray(self.m0, dtype=np.float64)
        self.m1 = np.asarray(self.m1, dtype=np.float64)
        if self.model not in (ADVECTION, CONTINUITY, INCOMPRESSIBLE):
            raise ValueError("model")
        if self.alpha <= 0:
            raise ValueError("alpha must be > 0")


def trapezoid_weights(nt: int):
    """w_0 = w_{n_t} = dt/2, w_j = dt otherwise (R10)."""
    dt = 1.0 / nt
    w = np.full(nt + 1, dt)
    w[0] = w[-1] = 0.5 * dt
    return w


def forward_solve(prob: Problem, v):
    """Feet, static factors and the state trajectory for velocity v."""
    g = prob.grid
    delta_f, delta_a = transport.feet(g, v, prob.nt)
    E_f = None
    if prob.model == CONTINUITY:
        E_f = transport.source_factor_forward_continuity(g, v, delta_f, prob.nt)
    traj = transport.forward(prob.m0, delta_f, prob.nt, E_f)
    return delta_f, delta_a, E_f, traj


def objective(prob: Problem, v):
    """obj(v) = dist + reg; forward solve only (what every Armijo trial needs)."""
    _, _, _, traj = forward_solve(prob, v)
    dist = 0.5 * spectral.inner(prob.grid, traj[-1] - prob.m1, traj[-1] - prob.m1)
    reg = spectral.reg_value(prob.grid, v, prob.alpha, prob.reg_order)
    return {"obj": dist + reg, "dist": dist, "reg": reg, "m_final": traj[-1]}


def evaluate(prob: Problem, v):
    """One objective-plus-gradient evaluation: forward, adjoint, body force, preconditioner.

    Returns a dict with every intermediate the GPU path exposes for parity:
    obj, dist, reg, delta_f, delta_a, E (static factor or None), m (trajectory),
    lam (trajectory), b (body force), g (reduced gradient), s (= -(alpha L~)^-1 g),
    grad_inf (= ||g||_inf), gs (= <g, s>_h).
    """
    grid = prob.grid
    v = np.asarray(v, dtype=np.float64)
    delta_f, delta_a, E_f, m = forward_solve(prob, v)
    mS = m[-1]
    dist = 0.5 * spectral.inner(grid, mS - prob.m1, mS - prob.m1)
    reg = spectral.reg_value(grid, v, prob.alpha, prob.reg_order)

    lam_final = prob.m1 - mS  # R1 (and R8 for continuity)
    E_a = None
    if prob.model == ADVECTION:
        E_a = transport.source_factor_adjoint_advection(grid, v, delta_a, prob.nt)
    lam = transport.adjoint(lam_final, delta_a, prob.nt, E_a)

    w = trapezoid_weights(prob.nt)
    b = np.zeros((grid.d,) + grid.shape)
    for j in range(prob.nt + 1):
        if prob.model == CONTINUITY:
            b -= w[j] * m[j] * spectral.grad(grid, lam[j])  # R8
        else:
            b += w[j] * lam[j] * spectral.grad(grid, m[j])  # (2.2)

    g = prob.alpha * spectral.apply_L(grid, v, prob.reg_order) + b
    if prob.model == INCOMPRESSIBLE:
        g = spectral.leray(grid, g)
    s = -spectral.apply_inv_alpha_L(grid, g, prob.alpha, prob.reg_order)
    return {
        "obj": dist + reg,
        "dist": dist,
        "reg": reg,
        "delta_f": delta_f,
        "delta_a": delta_a,
        "E": E_f if prob.model == CONTINUITY else E_a,
        "m": m,
        "lam": lam,
        "b": b,
        "g": g,
        "s": s,
        "grad_inf": float(np.max(np.abs(g))),
        "gs": spectral.inner(grid, g, s),
    }
