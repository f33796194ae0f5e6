"""Pins for oracle/flowmap.py (figure captions; reading R32):
identity, translations, a closed-form Jacobian, the characteristic identity for integer
shifts, and det -> 1 for divergence-free v under refinement."""
import numpy as np

from oracle import flowmap, spectral, transport
from oracle.spectral import Grid


def test_zero_velocity_identity():
    g = Grid((16, 12, 8))
    disp = flowmap.flow_map(g, np.zeros((3,) + g.shape), 4)
    assert np.all(disp == 0.0)
    assert np.all(flowmap.det_grad(g, disp) == 1.0)


def test_constant_velocity_is_a_translation():
    """Constant v: every foot is l - dt c/h and interpolating a constant is exact (partition
    of unity), so y - x = -c after n_t steps for ANY c, and det = 1."""
    g = Grid((32, 16))
    c = np.array([0.37, -0.21])
    v = np.stack([np.full(g.shape, ci) for ci in c])
    disp = flowmap.flow_map(g, v, 5)
    for a in range(2):
        np.testing.assert_allclose(disp[a], -c[a], atol=1e-13)
    np.testing.assert_allclose(flowmap.det_grad(g, disp), 1.0, atol=1e-13)


def test_det_grad_closed_form():
    """disp = (eps sin x1, eta sin x2): det = (1 + eps cos x1)(1 + eta cos x2) exactly."""
    g = Grid((32, 16, 8))
    x = g.coords()
    eps, eta = 0.3, -0.2
    disp = np.stack([eps * np.sin(x[0]), eta * np.sin(x[1]), np.zeros(g.shape)])
    np.testing.assert_allclose(flowmap.det_grad(g, disp), (1 + eps * np.cos(x[0])) * (1 + eta * np.cos(x[1])),
                               atol=1e-12)
    # a shear u1 = eps sin x2 has det 1 (off-diagonal only)
    disp = np.stack([eps * np.sin(x[1]), np.zeros(g.shape), np.zeros(g.shape)])
    np.testing.assert_allclose(flowmap.det_grad(g, disp), 1.0, atol=1e-12)


def test_characteristic_identity_integer_shift():
    """v dt/h an integer number of cells: the SL state m^S is an exact roll and so is
    I[m0](y)."""
    g = Grid((16, 16))
    nt = 4
    rng = np.random.default_rng(0)
    m0 = rng.normal(size=g.shape)
    cells = np.array([2.0, -1.0])
    v = np.stack([np.full(g.shape, cells[a] * g.h[a] * nt) for a in range(2)])
    disp = flowmap.flow_map(g, v, nt)
    df, _ = transport.feet(g, v, nt)
    mS = transport.forward(m0, df, nt)[-1]
    from oracle.interp import interp
    m_y = interp(m0, np.stack([disp[a] / g.h[a] for a in range(2)]))
    np.testing.assert_allclose(m_y, mS, atol=1e-12)
    # each step moves the foot by -cells: m^S(l) = m0(l - nt cells), numpy axes (x2, x1)
    shift = (int(nt * cells[1]), int(nt * cells[0]))
    np.testing.assert_allclose(m_y, np.roll(m0, shift=shift, axis=(0, 1)), atol=1e-12)


def test_divergence_free_det_tends_to_one():
    """Incompressible flow: det(grad y) = 1 for the exact map; the discrete map
    approaches it under refinement (n, n_t) -> (2n, 2n_t)."""
    errs = []
    for n, nt in ((64, 4), (128, 8)):
        g = Grid((n, n))
        x = g.coords()
        v = 0.2 * np.stack([np.sin(x[1]) * np.cos(x[0]), -np.sin(x[0]) * np.cos(x[1])])  # div v = 0
        det = flowmap.det_grad(g, flowmap.flow_map(g, v, nt))
        assert det.min() > 0.0
        errs.append(np.max(np.abs(det - 1.0)))
    assert errs[0] < 1e-3
    assert errs[1] < errs[0] / 2.0


def test_positive_determinant_for_config_velocity():
    """The paper's figures: det(grad y) > 0 (diffeomorphism) for the computed maps."""
    from synth import make_problem
    d = make_problem(1)
    g = Grid(tuple(d["n"]))
    det = flowmap.det_grad(g, flowmap.flow_map(g, d["vstar"], d["nt"]))
    assert det.min() > 0.0
