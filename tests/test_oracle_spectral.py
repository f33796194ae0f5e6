"""Pins for oracle/spectral.py against closed forms, brute-force DFT and invariants.

Paper passages: P:126-134 (Fourier grid, FFT operators, kernel fix of L),
P:29 / P:107 / P:734 (H2 biharmonic, H3 triharmonic), P:733-735 (div v = 0).
"""
import numpy as np
import pytest

from oracle import spectral
from oracle.spectral import Grid


def _brute_dft_deriv(f, a_axis_len, axis, n):
    """d/dx along numpy `axis` by an explicit O(n^2) DFT sum with k in (-n/2, n/2], Nyquist zeroed."""
    N = n
    l = np.arange(N)
    ks = np.arange(-N // 2 + 1, N // 2 + 1)  # R2 range
    E = np.exp(-1j * np.outer(ks, l) * 2 * np.pi / N)     # forward
    Einv = np.exp(1j * np.outer(l, ks) * 2 * np.pi / N) / N
    sym = 1j * ks.astype(float)
    sym[ks == N // 2] = 0.0                                 # R3
    fm = np.moveaxis(f, axis, -1)
    out = np.real(((fm @ E.T) * sym) @ Einv.T)
    return np.moveaxis(out, -1, axis)


def test_deriv_matches_bruteforce_dft():
    rng = np.random.default_rng(1)
    g = Grid((8, 6))
    f = rng.normal(size=g.shape)
    for a in range(2):
        ref = _brute_dft_deriv(f, g.n[a], g.axis(a), g.n[a])
        np.testing.assert_allclose(spectral.deriv(g, f, a), ref, atol=1e-12)


def test_deriv_single_modes_exact():
    g = Grid((32, 16, 8))
    x1, x2, x3 = g.coords()
    f = np.sin(3 * x1) * np.cos(2 * x2) * np.cos(x3)
    np.testing.assert_allclose(spectral.deriv(g, f, 0), 3 * np.cos(3 * x1) * np.cos(2 * x2) * np.cos(x3), atol=1e-12)
    np.testing.assert_allclose(spectral.deriv(g, f, 1), -2 * np.sin(3 * x1) * np.sin(2 * x2) * np.cos(x3), atol=1e-12)
    np.testing.assert_allclose(spectral.deriv(g, f, 2), -np.sin(3 * x1) * np.cos(2 * x2) * np.sin(x3), atol=1e-12)


def test_nyquist_zeroed_in_odd_derivative():
    """Reading R3: the Nyquist mode cos(n/2 x) has zero derivative (keeps real fields real)."""
    g = Grid((16, 16))
    x1, _ = g.coords()
    assert np.max(np.abs(spectral.deriv(g, np.cos(8 * x1), 0))) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3])
def test_L_eigenvalue_single_mode(p):
    """sin(k.x) is an eigenfunction of L with eigenvalue |k|^{2p} (R4)."""
    g = Grid((16, 16, 16))
    x1, x2, x3 = g.coords()
    k = (3, -2, 1)
    mode = np.sin(k[0] * x1 + k[1] * x2 + k[2] * x3 + 0.4)
    u = np.stack([mode, 0 * mode, 0 * mode])
    Lu = spectral.apply_L(g, u, p)
    np.testing.assert_allclose(Lu[0], (9 + 4 + 1) ** p * mode, atol=1e-9 * 14 ** p)
    # Nyquist uses the true wavenumber n/2 in L (R3): cos(8 x1) -> 8^{2p}
    ny = np.cos(8 * x1)
    np.testing.assert_allclose(spectral.apply_L(g, np.stack([ny, ny, ny]), p)[1], 8.0 ** (2 * p) * ny,
                               rtol=1e-10, atol=1e-9)


def test_golden_reg_symbols():
    """tests/golden/reg_symbol.txt: |k|^{2p} values (SPEC S:67-69 worked examples)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "reg_symbol.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    assert rows
    for p, k1, k2, expect in rows:
        g = Grid((16, 16))
        sym = spectral.reg_symbol(g, int(p))
        assert sym[int(k2) % 16, int(k1) % 16] == float(expect)


def test_inverse_regularisation_closed_form():
    """(alpha L~)^{-1} mode = mode / (alpha |k|^{2p}); the mean is divided by alpha (kernel fix)."""
    g = Grid((16, 16))
    x1, x2 = g.coords()
    alpha = 0.1
    mode = 2.0 * np.sin(x1)
    out = spectral.apply_inv_alpha_L(g, np.stack([mode, 0 * mode + 3.0]), alpha, 2)
    np.testing.assert_allclose(out[0], mode / alpha, atol=1e-12)
    np.testing.assert_allclose(out[1], 3.0 / alpha, atol=1e-12)
    # L (alpha L~)^{-1} = 1/alpha on the complement of the kernel
    rng = np.random.default_rng(3)
    u = rng.normal(size=(2,) + g.shape)
    u -= u.mean(axis=(1, 2), keepdims=True)
    back = alpha * spectral.apply_L(g, spectral.apply_inv_alpha_L(g, u, alpha, 2), 2)
    np.testing.assert_allclose(back, u, atol=1e-10)


def test_reg_value_parseval_closed_form():
    """alpha/2 <v, L v>_h for v = a sin(k.x) e_1 equals alpha/2 |k|^{2p} a^2 (2pi)^d / 2."""
    g = Grid((32, 32))
    x1, x2 = g.coords()
    a, alpha = 0.7, 0.3
    v = np.stack([a * np.sin(2 * x1 - 3 * x2), 0 * x1])
    for p in (1, 2, 3):
        ref = 0.5 * alpha * 13 ** p * a * a * (2 * np.pi) ** 2 / 2
        assert abs(spectral.reg_value(g, v, alpha, p) - ref) < 1e-10 * ref


def test_integration_by_parts():
    """<grad f, u>_h = -<f, div u>_h on random fields."""
    rng = np.random.default_rng(4)
    g = Grid((12, 10, 8))
    f = rng.normal(size=g.shape)
    u = rng.normal(size=(3,) + g.shape)
    lhs = spectral.inner(g, spectral.grad(g, f), u)
    rhs = -spectral.inner(g, f, spectral.div(g, u))
    assert abs(lhs - rhs) < 1e-11 * (abs(lhs) + 1)


def test_leray_properties():
    """Leray projector: div-free output, idempotent, self-adjoint, kills gradients, fixes curls (R3, R9)."""
    rng = np.random.default_rng(5)
    for n in ((64, 64), (16, 12, 8)):
        g = Grid(n)
        u = rng.normal(size=(g.d,) + g.shape)
        w = rng.normal(size=(g.d,) + g.shape)
        Pu = spectral.leray(g, u)
        assert np.max(np.abs(spectral.div(g, Pu))) < 1e-10
        np.testing.assert_allclose(spectral.leray(g, Pu), Pu, atol=1e-12)
        assert abs(spectral.inner(g, Pu, w) - spectral.inner(g, u, spectral.leray(g, w))) < 1e-10
        f = rng.normal(size=g.shape)
        assert np.max(np.abs(spectral.leray(g, spectral.grad(g, f)))) < 1e-10
    g = Grid((32, 32))
    x1, x2 = g.coords()
    psi = np.sin(2 * x1) * np.cos(3 * x2)
    curl = np.stack([-spectral.deriv(g, psi, 1), spectral.deriv(g, psi, 0)])
    np.testing.assert_allclose(spectral.leray(g, curl), curl, atol=1e-12)


def test_gaussian_blur_mode():
    g = Grid((64, 64))
    x1, _ = g.coords()
    out = spectral.gaussian_blur(g, np.sin(x1), 1.0)
    np.testing.assert_allclose(out, np.exp(-0.5 * (2 * np.pi / 64) ** 2) * np.sin(x1), atol=1e-14)


def test_dft_coeff_closed_form():
    """f = cos(k0 . x + phi): f^_{k0} = (N/2) e^{i phi}, f^_{-k0} = (N/2) e^{-i phi}, 0 elsewhere."""
    g = Grid((8, 6, 4))
    x = g.coords()
    k0, phi = (3, -2, 1), 0.7
    f = np.cos(sum(k * xa for k, xa in zip(k0, x)) + phi)
    N = g.npts
    assert abs(spectral.dft_coeff(g, f, k0) - 0.5 * N * np.exp(1j * phi)) < 1e-10 * N
    assert abs(spectral.dft_coeff(g, f, tuple(-k for k in k0)) - 0.5 * N * np.exp(-1j * phi)) < 1e-10 * N
    for k in [(0, 0, 0), (3, 2, 1), (1, -2, 1), (3, -2, -1)]:
        assert abs(spectral.dft_coeff(g, f, k)) < 1e-10 * N
    # a constant: f^_0 = N c
    assert abs(spectral.dft_coeff(g, np.full(g.shape, 2.5), (0, 0, 0)) - 2.5 * N) < 1e-10 * N


def test_deriv_line_modes_and_nyquist():
    n = 32
    x = np.arange(n) * 2 * np.pi / n
    np.testing.assert_allclose(spectral.deriv_line(np.sin(3 * x + 0.4)), 3 * np.cos(3 * x + 0.4), atol=1e-12)
    np.testing.assert_allclose(spectral.deriv_line(np.cos(15 * x)), -15 * np.sin(15 * x), atol=1e-11)
    assert np.max(np.abs(spectral.deriv_line(np.cos(16 * x)))) < 1e-12  # Nyquist zeroed (R3)
    # rows of a 2D array are independent lines; brute-force O(n^2) DFT on random data
    rng = np.random.default_rng(3)
    f = rng.normal(size=(3, 16))
    np.testing.assert_allclose(spectral.deriv_line(f), _brute_dft_deriv(f, 16, 1, 16), atol=1e-11)
