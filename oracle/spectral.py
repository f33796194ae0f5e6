"""Fourier pseudo-spectral layer of the oracle (fp64).  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2.2 "Numerical Discretization":
  * Omega = [0, 2pi)^d, n_i cells per axis, h_i = 2pi/n_i, nodes x_l = 2pi l (/) n
  * u(x) = sum_k u_k exp(i <k, x>), -n_j/2+1 <= k_j <= n_j/2   (reading R2: the
    printed lower bound lost its minus sign)
  * derivatives/operators applied "at the cost of two FFTs and a diagonal
    scaling"; zero spectral entries of L are set to one before inverting

Readings: R2 wavenumber range, R3 odd derivatives zero the
Nyquist index (and the Leray projector uses the same k'), R4 L(k)=|k|^(2p),
R11 discrete inner product <a,b>_h = h^d sum a*b.

Array layout: a scalar field has numpy shape (n_d, ..., n_1) — C order with
x_1 fastest; a vector field has shape (d, n_d, ..., n_1) with component c the
x_{c+1} component.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np


@dataclass(frozen=True)
class Grid:
    """Periodic grid on [0, 2pi)^d.  ``n`` is given in paper order (n_1, ..., n_d)."""

    n: tuple

    def __post_init__(self):
        if len(self.n) not in (2, 3):
            raise ValueError("d must be 2 or 3")
        for ni in self.n:
            if ni < 4 or ni % 2:
                raise ValueError("n_i must be even and >= 4")

    @property
    def d(self) -> int:
        return len(self.n)

    @property
    def shape(self) -> tuple:
        """numpy shape of a scalar field: (n_d, ..., n_1)."""
        return tuple(reversed(self.n))

    @property
    def h(self) -> tuple:
        """Mesh sizes h_i = 2pi/n_i in paper order."""
        return tuple(2.0 * np.pi / ni for ni in self.n)

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.h))

    @property
    def npts(self) -> int:
        return int(np.prod(self.n))

    def axis(self, a: int) -> int:
        """numpy axis of paper axis a (0-based: a=0 is x_1)."""
        return self.d - 1 - a

    def coords(self):
        """Node coordinates x_l = 2pi l / n, as a list [x_1, ..., x_d] of full arrays."""
        g = [np.arange(ni) * (2.0 * np.pi / ni) for ni in self.n]
        mesh = np.meshgrid(*reversed(g), indexing="ij")  # numpy order
        return list(reversed(mesh))

    @cached_property
    def k(self):
        """Integer wavenumbers per paper axis, broadcast to the spectral array shape.

        np.fft ordering; index n_j/2 carries k_j = -n_j/2, identified with +n_j/2
        (R2) — only k_j^2 (for L) or the Nyquist-zeroed k' (odd operators) are used.
        """
        out = []
        for a, ni in enumerate(self.n):
            ka = np.fft.fftfreq(ni, d=1.0 / ni)
            shp = [1] * self.d
            shp[self.axis(a)] = ni
            out.append(ka.reshape(shp))
        return out

    @cached_property
    def kprime(self):
        """k' : wavenumbers with the Nyquist index zeroed (reading R3)."""
        out = []
        for a, ni in enumerate(self.n):
            ka = np.fft.fftfreq(ni, d=1.0 / ni)
            ka[ni // 2] = 0.0
            shp = [1] * self.d
            shp[self.axis(a)] = ni
            out.append(ka.reshape(shp))
        return out

    @cached_property
    def ksq(self):
        """|k|^2 with the true Nyquist value (R3, R4)."""
        s = 0.0
        for ka in self.k:
            s = s + ka * ka
        return s


def fft(u):
    return np.fft.fftn(u)


def ifft_real(uh):
    return np.real(np.fft.ifftn(uh))


def deriv(grid: Grid, f, a: int):
    """Spectral derivative d/dx_{a+1} of a scalar field: symbol i k'_a (R3)."""
    return ifft_real(1j * grid.kprime[a] * fft(f))


def grad(grid: Grid, f):
    """Spectral gradient, shape (d, *shape)."""
    return np.stack([deriv(grid, f, a) for a in range(grid.d)])


def div(grid: Grid, u):
    """Spectral divergence sum_a d u_a / dx_a (Nyquist zeroed, R3)."""
    return sum(deriv(grid, u[a], a) for a in range(grid.d))


def reg_symbol(grid: Grid, p: int):
    """L(k) = |k|^{2p}: H1 -> |k|^2, H2 (biharmonic) -> |k|^4, H3 -> |k|^6 (R4)."""
    if p not in (1, 2, 3):
        raise ValueError("regularisation order p must be 1, 2 or 3")
    return grid.ksq ** p


def reg_symbol_fixed(grid: Grid, p: int):
    """L~(k): zero entries of L set to one before inversion."""
    L = reg_symbol(grid, p)
    return np.where(L == 0.0, 1.0, L)


def apply_L(grid: Grid, u, p: int):
    """L u for a vector field (componentwise)."""
    L = reg_symbol(grid, p)
    return np.stack([ifft_real(L * fft(u[c])) for c in range(u.shape[0])])


def apply_inv_alpha_L(grid: Grid, u, alpha: float, p: int):
    """(alpha L~)^{-1} u componentwise: "two FFTs and a diagonal scaling", kernel fix."""
    Lt = reg_symbol_fixed(grid, p)
    return np.stack([ifft_real(fft(u[c]) / (alpha * Lt)) for c in range(u.shape[0])])


def leray(grid: Grid, u):
    """Leray projector P_L u = u - k'(k'.u)/|k'|^2 for k' != 0, unchanged for k' = 0 (R3, R9)."""
    uh = [fft(u[c]) for c in range(grid.d)]
    kp = grid.kprime
    kk = sum(kp[a] * kp[a] for a in range(grid.d))
    dot = sum(kp[a] * uh[a] for a in range(grid.d))
    safe = np.where(kk == 0.0, 1.0, kk)
    coef = np.where(kk == 0.0, 0.0, dot / safe)
    return np.stack([ifft_real(uh[a] - kp[a] * coef) for a in range(grid.d)])


def inner(grid: Grid, a, b) -> float:
    """Discrete L2 inner product <a,b>_h = h^d sum a*b (reading R11)."""
    return float(grid.cell_volume * np.sum(a * b))


def reg_value(grid: Grid, v, alpha: float, p: int) -> float:
    """(alpha/2) <v, L v>_h: the regularisation term of (1.1a) (reading R23)."""
    return 0.5 * alpha * inner(grid, v, apply_L(grid, v, p))


def dft_coeff(grid: Grid, f, kvec) -> complex:
    """One DFT coefficient f^_k = sum_l f_l exp(-i k . x_l), x_l = 2 pi l / n (R2), by
    its plain definition, one axis at a time.  The phase k x_l = 2 pi ((k l) mod n) / n is
    reduced in integers, so it is exact before the cos / sin (a high |k| times an inexact
    x_l would carry a phase error that alpha |k|^{2p} amplifies).  kvec: integer
    wavenumbers in paper order.  Used to check full-size spectral outputs at sampled modes."""
    out = np.asarray(f)
    for a in range(grid.d):  # paper axis a = numpy axis d-1-a; contract the last one each time
        na = grid.n[a]
        m = (int(kvec[a]) * np.arange(na, dtype=np.int64)) % na
        ang = 2.0 * np.pi * m / na
        if np.iscomplexobj(out):
            out = out @ (np.cos(ang) - 1j * np.sin(ang))
        else:  # real field: first contraction in real arithmetic (cos and sin parts)
            out = (out.astype(np.float64) @ np.cos(ang)) - 1j * (out.astype(np.float64) @ np.sin(ang))
    return complex(out)


def deriv_line(f_line):
    """Spectral derivative of one periodic line on [0, 2pi): symbol i k' with the Nyquist
    index zeroed (R3).  Used to check full-size derivative outputs on sampled lines."""
    f_line = np.asarray(f_line, dtype=np.float64)
    n = f_line.shape[-1]
    k = np.fft.fftfreq(n, d=1.0 / n)
    k[n // 2] = 0.0
    return np.real(np.fft.ifft(1j * k * np.fft.fft(f_line, axis=-1), axis=-1))


def gaussian_blur(grid: Grid, f, sigma_vox: float):
    """Spectral Gaussian smoothing with std sigma_vox*h_i.  Used by pins only."""
    mult = 1.0
    for a in range(grid.d):
        s = sigma_vox * grid.h[a]
        mult = mult * np.exp(-0.5 * (s * grid.k[a]) ** 2)
    return ifft_real(mult * fft(f))
