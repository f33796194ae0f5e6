"""Semi-Lagrangian transport solves (fp64).  TEST INFRASTRUCTURE ONLY.

PAPER.md anchors:
  * state equation (1.1b)  d_t m + grad m . v = 0, m(0) = m0
  * adjoint (2.3)          -d_t lam - div(lam v) = 0, terminal at t=1
  * continuity (3.1b)      d_t pi + div(pi v) = 0, pi(0) = pi0
  * "semi-Lagrangian scheme ... unconditionally stable ... explicit,
    second-order Runge-Kutta"; n_t cells of size h_t = 1/n_t

Readings:
  R5  positions are node + displacement in cells, tricubic Lagrange interpolant
  R6  RK2 = midpoint rule for the characteristic trace:
        forward foot  X = x - dt v(x - dt/2 v(x))
        adjoint foot  Y = x + dt v(x + dt/2 v(x))
      v is stationary, so the feet are static over all n_t steps.
  R7  conservative source terms (adjoint of A, forward of C) are integrated with
      Heun's rule along the characteristic using the divergence at the foot
      (a) and at the arrival node (b):
        C forward:  pi^{j+1} = I[pi^j](X) * (1 - dt/2 (a+b) + dt^2/2 a b)
        A adjoint:  lam^j    = I[lam^{j+1}](Y) * (1 + dt/2 (a'+b) + dt^2/2 a' b)
  R8  continuity adjoint is pure advection: -d_t lam - v.grad lam = 0
  R9  incompressible: v divergence free, the A adjoint with factor 1
"""
from __future__ import annotations

import numpy as np

from . import spectral
from .interp import interp, interp_vec

ADVECTION, CONTINUITY, INCOMPRESSIBLE = 0, 1, 2


def velocity_in_cells(grid: spectral.Grid, v):
    """v_a / h_a : velocity in cells per unit time."""
    return np.stack([v[a] / grid.h[a] for a in range(grid.d)])


def feet(grid: spectral.Grid, v, nt: int):
    """Midpoint-RK2 characteristic feet as displacements in cells (R5, R6).

    Returns (delta_f, delta_a), each shape (d, *shape):
      delta_f = -dt * I[v/h](l - dt/2 * v_l/h)     (forward foot  X - x)
      delta_a = +dt * I[v/h](l + dt/2 * v_l/h)     (adjoint foot  Y - x)
    """
    dt = 1.0 / nt
    vc = velocity_in_cells(grid, v)
    delta_f = -dt * interp_vec(vc, -0.5 * dt * vc)
    delta_a = dt * interp_vec(vc, 0.5 * dt * vc)
    return delta_f, delta_a


def source_factor_forward_continuity(grid, v, delta_f, nt):
    """E_f = 1 - dt/2 (a + b) + dt^2/2 a b, a = div v at the forward foot, b = div v (R7)."""
    dt = 1.0 / nt
    b = spectral.div(grid, v)
    a = interp(b, delta_f)
    return 1.0 - 0.5 * dt * (a + b) + 0.5 * dt * dt * a * b


def source_factor_adjoint_advection(grid, v, delta_a, nt):
    """E_a = 1 + dt/2 (a' + b) + dt^2/2 a' b, a' = div v at the adjoint foot (R7)."""
    dt = 1.0 / nt
    b = spectral.div(grid, v)
    a = interp(b, delta_a)
    return 1.0 + 0.5 * dt * (a + b) + 0.5 * dt * dt * a * b


def forward(m0, delta_f, nt: int, factor=None):
    """State trajectory [m^0, ..., m^{n_t}] : m^{j+1} = I[m^j](l + delta_f) (* E_f for C)."""
    traj = [np.array(m0, dtype=np.float64)]
    for _ in range(nt):
        nxt = interp(traj[-1], delta_f)
        if factor is not None:
            nxt = nxt * factor
        traj.append(nxt)
    return traj


def adjoint(lam_final, delta_a, nt: int, factor=None):
    """Adjoint trajectory [lam^0, ..., lam^{n_t}], integrated backward from lam^{n_t}."""
    traj = [None] * (nt + 1)
    traj[nt] = np.array(lam_final, dtype=np.float64)
    for j in range(nt - 1, -1, -1):
        nxt = interp(traj[j + 1], delta_a)
        if factor is not None:
            nxt = nxt * factor
        traj[j] = nxt
    return traj
