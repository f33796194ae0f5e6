"""Pins for oracle/interp.py and oracle/transport.py.

Paper passages: P:35-41 (state equation), P:110-121 (adjoint)
(continuity), P:136 (unconditionally stable SL with RK2); readings R5-R8.
"""
import numpy as np
import pytest
import torch

from oracle import interp as I
from oracle import spectral, transport
from oracle.spectral import Grid
from synth.phantoms import sample_sinusoid_field


def _field_from(g, sf):
    X = torch.tensor(np.stack([c.ravel() for c in g.coords()]))
    v, div = sf.eval(X)
    return v.numpy().reshape((g.d,) + g.shape), div.numpy().reshape(g.shape)


def _smooth(g, seed=0):
    rng = np.random.default_rng(seed)
    return spectral.gaussian_blur(g, rng.normal(size=g.shape), 3.0)


# ---------------------------------------------------------------- interpolation (R5)
@pytest.mark.parametrize("t", [0.0, 0.1, 0.37, 0.5, 0.99])
def test_lagrange_weights_reproduce_cubics(t):
    """Cubic Lagrange weights on nodes -1..2 reproduce 1, s, s^2, s^3 at s = t."""
    w = np.array(I.lagrange_weights(t))
    nodes = np.array([-1.0, 0.0, 1.0, 2.0])
    for m in range(4):
        assert abs(w @ nodes ** m - t ** m) < 1e-14


def test_interp_reproduces_local_cubic_3d():
    """Tensor-product cubic polynomial is reproduced exactly away from the periodic seam."""
    g = Grid((16, 16, 16))
    l3, l2, l1 = np.meshgrid(*(np.arange(16.0),) * 3, indexing="ij")
    f = (l1 - 3.3) ** 3 * (l2 - 7.1) ** 2 * (l3 + 0.5) + 2.0 * l2 - l3 ** 3
    rng = np.random.default_rng(2)
    delta = rng.uniform(-1.5, 1.5, size=(3,) + g.shape)
    out = I.interp(f, delta)
    inner = (slice(4, 12),) * 3
    p1, p2, p3 = l1 + delta[0], l2 + delta[1], l3 + delta[2]
    ref = (p1 - 3.3) ** 3 * (p2 - 7.1) ** 2 * (p3 + 0.5) + 2.0 * p2 - p3 ** 3
    np.testing.assert_allclose(out[inner], ref[inner], rtol=1e-11, atol=1e-9)


def test_interp_nodes_and_periodic_wrap():
    g = Grid((8, 6, 4))
    rng = np.random.default_rng(3)
    f = rng.normal(size=g.shape)
    zero = np.zeros((3,) + g.shape)
    assert np.array_equal(I.interp(f, zero), f)                       # nodes: exact, bitwise
    shift = zero.copy(); shift[0] += 8; shift[1] -= 12; shift[2] += 4
    assert np.array_equal(I.interp(f, shift), f)                      # full periods
    one = zero.copy(); one[0] += 1.0; one[2] -= 1.0
    np.testing.assert_array_equal(I.interp(f, one), np.roll(np.roll(f, -1, axis=2), 1, axis=0))


def test_interp_fourth_order_convergence():
    errs = []
    for n in (32, 64, 128):
        g = Grid((n, n))
        x1, x2 = g.coords()
        d = np.stack([0.3 + 0 * x1, -0.45 + 0 * x1])
        out = I.interp(np.sin(x1) * np.cos(2 * x2), d)
        h = 2 * np.pi / n
        errs.append(np.max(np.abs(out - np.sin(x1 + 0.3 * h) * np.cos(2 * (x2 - 0.45 * h)))))
    assert errs[0] / errs[1] > 12 and errs[1] / errs[2] > 12


# ---------------------------------------------------------------- forward sweep
def test_zero_velocity_is_identity_bitwise():
    g = Grid((16, 16, 8))
    m0 = _smooth(g)
    df, da = transport.feet(g, np.zeros((3,) + g.shape), 4)
    assert not df.any() and not da.any()
    traj = transport.forward(m0, df, 4)
    for m in traj:
        assert np.array_equal(m, m0)


@pytest.mark.parametrize("n,c", [((64, 64), (0.37, -0.21)), ((32, 16, 24), (0.5, 0.9, -1.3))])
def test_constant_velocity_mode_closed_form(n, c):
    """Constant v: the discrete scheme is diagonal in Fourier space; m^S = mu(k)^S e^{ik.x} with
    mu = prod_a e^{i k_a h_a floor(d_a)} sum_j w_{j-1}(t_a) e^{i k_a h_a (j-1)},  d = -dt c/h."""
    g = Grid(n)
    nt = 4
    dt = 1.0 / nt
    k = (3, -2, 1)[: g.d]
    xs = g.coords()
    phase = sum(k[a] * xs[a] for a in range(g.d))
    v = np.stack([np.full(g.shape, c[a]) for a in range(g.d)])
    df, _ = transport.feet(g, v, nt)
    traj = transport.forward(np.cos(phase + 0.3), df, nt)
    mu = 1.0 + 0j
    for a in range(g.d):
        d = -dt * c[a] / g.h[a]
        fl = np.floor(d)
        t = d - fl
        w = I.lagrange_weights(t)
        kh = k[a] * g.h[a]
        mu *= np.exp(1j * kh * fl) * sum(w[j] * np.exp(1j * kh * (j - 1)) for j in range(4))
    ref = np.real(mu ** nt * np.exp(1j * (phase + 0.3)))
    np.testing.assert_allclose(traj[-1], ref, atol=1e-13)


def test_integer_cell_velocity_is_exact_translation():
    """c dt / h integer => exact periodic translation (BASELINE 'equals the exact translation')."""
    g = Grid((32, 16, 8))
    nt = 4
    m0 = _smooth(g, 1)
    cells = (2, -1, 3)
    v = np.stack([np.full(g.shape, cells[a] * g.h[a] * nt) for a in range(3)])
    df, _ = transport.feet(g, v, nt)
    out = transport.forward(m0, df, nt)[-1]
    ref = m0
    for a in range(3):
        ref = np.roll(ref, nt * cells[a], axis=g.axis(a))
    np.testing.assert_allclose(out, ref, atol=1e-12)


def test_sl_unconditionally_stable_large_cfl():
    """P:136 'unconditionally stable': 16 cells per step keeps max|m| bounded."""
    g = Grid((64, 64))
    m0 = _smooth(g, 2)
    v = np.stack([np.full(g.shape, 16 * g.h[0] * 4 + 0.013), np.full(g.shape, -0.7)])
    df, _ = transport.feet(g, v, 4)
    out = transport.forward(m0, df, 4)[-1]
    assert np.max(np.abs(out)) <= 1.01 * np.max(np.abs(m0))


# ---------------------------------------------------------------- continuity / adjoint (R7, R8)
def test_continuity_constant_velocity_conserves_mass_exactly():
    g = Grid((32, 32, 16))
    m0 = np.abs(_smooth(g, 4))
    v = np.stack([np.full(g.shape, x) for x in (0.31, -0.52, 0.77)])
    df, _ = transport.feet(g, v, 4)
    E = transport.source_factor_forward_continuity(g, v, df, 4)
    np.testing.assert_allclose(E, 1.0, atol=1e-13)
    out = transport.forward(m0, df, 4, E)[-1]
    assert abs(out.sum() - m0.sum()) < 1e-12 * m0.sum()


def test_continuity_mass_drift_small_and_factor_sign():
    """General compressible v: relative mass drift <= 1e-3; a flipped source sign fails."""
    g = Grid((64, 64))
    rng = np.random.Generator(np.random.PCG64(7))
    v, _ = _field_from(g, sample_sinusoid_field(rng, 2, 2, 2, 0.15))
    m0 = np.abs(_smooth(g, 5)) + 0.1
    df, _ = transport.feet(g, v, 4)
    E = transport.source_factor_forward_continuity(g, v, df, 4)
    drift = abs(transport.forward(m0, df, 4, E)[-1].sum() / m0.sum() - 1)
    wrong = abs(transport.forward(m0, df, 4, 2.0 - E)[-1].sum() / m0.sum() - 1)
    assert drift < 1e-3 and wrong > 20 * drift


def test_continuity_equals_advection_for_divergence_free_v():
    g = Grid((32, 32))
    rng = np.random.Generator(np.random.PCG64(8))
    v, div = _field_from(g, sample_sinusoid_field(rng, 2, 2, 3, 0.3, divfree=True))
    assert np.max(np.abs(div)) < 1e-14
    m0 = _smooth(g, 6)
    df, _ = transport.feet(g, v, 4)
    E = transport.source_factor_forward_continuity(g, v, df, 4)
    np.testing.assert_allclose(transport.forward(m0, df, 4, E)[-1], transport.forward(m0, df, 4)[-1],
                               atol=1e-12)


def test_adjoint_zero_velocity_and_zero_residual():
    g = Grid((16, 16))
    m0, m1 = _smooth(g, 1), _smooth(g, 2)
    zero = np.zeros((2,) + g.shape)
    _, da = transport.feet(g, zero, 4)
    E = transport.source_factor_adjoint_advection(g, zero, da, 4)
    lam = transport.adjoint(m1 - m0, da, 4, E)
    for l in lam:
        assert np.array_equal(l, m1 - m0)
    lam0 = transport.adjoint(np.zeros(g.shape), da, 4, E)
    assert all(not l.any() for l in lam0)


def test_adjoint_duality_advection():
    """<m^S, lam^S>_h ~= <m^0, lam^0>_h (d/dt <m, lam> = 0 in the continuum); a flipped
    adjoint source factor (R7) breaks it by an order of magnitude."""
    g = Grid((64, 64))
    rng = np.random.Generator(np.random.PCG64(7))
    v, _ = _field_from(g, sample_sinusoid_field(rng, 2, 2, 2, 0.3))
    m0, lamS = _smooth(g, 1), _smooth(g, 2)
    df, da = transport.feet(g, v, 4)
    E = transport.source_factor_adjoint_advection(g, v, da, 4)
    m = transport.forward(m0, df, 4)

    def err(fac):
        lam = transport.adjoint(lamS, da, 4, fac)
        a, b = spectral.inner(g, m[-1], lam[-1]), spectral.inner(g, m[0], lam[0])
        return abs(a - b) / abs(a)

    assert err(E) < 2e-2 and err(2.0 - E) > 5 * err(E)


def test_interp_at_equals_field_interp_at_the_same_nodes():
    """Point-list interpolation = the whole-field routine (pinned above) at those nodes."""
    from oracle.interp import interp, interp_at
    rng = np.random.default_rng(7)
    f = rng.normal(size=(8, 12, 16))
    delta = rng.uniform(-3.5, 3.5, size=(3,) + f.shape)
    full = interp(f, delta)
    idx = rng.integers(0, 8 * 12 * 16, size=50)
    k, j, i = np.unravel_index(idx, f.shape)
    nodes = np.stack([i, j, k])
    got = interp_at(f, nodes, delta[:, k, j, i])
    np.testing.assert_array_equal(got, full[k, j, i])
