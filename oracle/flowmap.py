"""Flow-map diagnostics: the map y and det(grad y) (fp64).  TEST INFRASTRUCTURE ONLY.

PAPER.md anchors: the figure captions P:323, P:781, P:866 show "the computed mapping y" and
"the determinant of the deformation gradient (the values are all positive, illustrating
that the computed map y is a diffeomorphism)"; for the incompressible model the
determinant "is equal to 1 to high accuracy".  The paper gives no construction; reading R32
(SPEC S:210-227 as interface reference):

  * y(x) is the foot at t = 0 of the characteristic that ends at x at t = 1.  With the
    stationary v and the static RK2 forward foot X = l + delta_f(l) (R5, R6), the discrete
    map is the composition of the n_t one-step backward maps: the displacement u = y - x
    (periodic, in cells) obeys
        u^0 = 0,   u^{j+1}(l) = delta_f(l) + I[u^j](l + delta_f(l)),   u = u^{n_t};
  * det(grad y) = det(I + grad u), with grad u by spectral differentiation of the periodic
    displacement (R3) in physical units (u_b h_b).
"""
from __future__ import annotations

import numpy as np

from . import spectral, transport
from .interp import interp_vec


def flow_map(grid: spectral.Grid, v, nt: int):
    """Displacement y(x) - x in physical units (radians), shape (d, *shape)."""
    delta_f, _ = transport.feet(grid, v, nt)
    u = np.zeros_like(delta_f)
    for _ in range(nt):
        u = delta_f + interp_vec(u, delta_f)
    return np.stack([u[b] * grid.h[b] for b in range(grid.d)])


def det_grad(grid: spectral.Grid, disp):
    """det(I + grad disp), disp = y - x in radians (d, *shape)."""
    d = grid.d
    J = [[(1.0 if a == b else 0.0) + spectral.deriv(grid, disp[b], a) for a in range(d)] for b in range(d)]
    if d == 2:
        return J[0][0] * J[1][1] - J[0][1] * J[1][0]
    return (J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
            - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
            + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]))
