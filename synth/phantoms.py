"""Seeded synthetic problems (BASELINE.json configs 1-5).  No method arithmetic here.

Every field is a closed form evaluated at grid nodes (or at the exact
characteristic foot Phi^{-1}(x) for m1).  Parameters are drawn from
numpy.random.Generator(PCG64(2510087820 + config)) in the order written below.
Evaluation runs in torch fp64 on any device (large configs are generated on
the GPU by bench.py; the results are the same closed forms either way).

Stand-ins: the paper's data (hands, nirep, rect, smooth
sinusoids, Gaussian densities) are not available; these
smooth phantoms follow BASELINE.json's recipe instead.  "Gaussian blur sigma=s
voxels" is realised analytically as an erfc edge of width s*h across the
(approximate) signed distance to each ellipsoid surface.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

SEED0 = 2510087820
TWO_PI = 2.0 * math.pi

# Solver / model settings of the five BASELINE.json configs (readings R14, R27-R29).
CONFIGS = {
    1: dict(n=(64, 64), model=0, nt=4, reg_order=2, alpha=1e-2, window=5, sigma=1, tau=2,
            max_iter=20, eps_rel=5e-2),
    2: dict(n=(64, 64, 64), model=0, nt=4, reg_order=1, alpha=1e-2, window=5, sigma=1, tau=0,
            max_iter=20, eps_rel=5e-2),
    3: dict(n=(128, 128, 128), model=2, nt=8, reg_order=2, alpha=1e-3, window=5, sigma=1, tau=0,
            max_iter=20, eps_rel=5e-2),
    4: dict(n=(256, 256, 256), model=1, nt=8, reg_order=2, alpha=1e-3, window=5, sigma=1, tau=0,
            max_iter=20, eps_rel=5e-2),
    5: dict(n=(512, 512, 512), model=0, nt=16, reg_order=2, alpha=1e-3, window=10, sigma=1,
            tau=0, max_iter=20, eps_rel=5e-2),
}


@dataclass
class SinusoidField:
    """v(X) = sum_m a_m sin(k_m . X + phi_m); k_m integer (d,), a_m real (d,)."""

    k: np.ndarray      # (M, d)
    phi: np.ndarray    # (M,)
    a: np.ndarray      # (M, d)
    scale: float = 1.0

    def eval(self, X):
        """X: tensor (d, N) -> (v (d, N), div v (N,))."""
        k = torch.as_tensor(self.k, dtype=X.dtype, device=X.device)
        a = torch.as_tensor(self.a, dtype=X.dtype, device=X.device) * self.scale
        phi = torch.as_tensor(self.phi, dtype=X.dtype, device=X.device)
        arg = k @ X + phi[:, None]                      # (M, N)
        s, c = torch.sin(arg), torch.cos(arg)
        v = a.T @ s                                     # (d, N)
        div = ((a * k).sum(dim=1)[:, None] * c).sum(0)  # sum_m (a_m.k_m) cos
        return v, div


def _random_k(rng, d, kmax):
    """Integer k with 1 <= |k|_2 <= kmax, rejection from [-kmax, kmax]^d."""
    while True:
        k = rng.integers(-kmax, kmax + 1, size=d)
        r = float(np.sqrt((k * k).sum()))
        if 1.0 <= r <= kmax:
            return k


def sample_sinusoid_field(rng, d, per_component, kmax, amplitude, divfree=False):
    """Seeded random sinusoid velocity; amplitude is a per-mode factor (unscaled)."""
    ks, phis, amps = [], [], []
    if divfree:
        for _ in range(per_component * d):
            k = _random_k(rng, d, kmax)
            e = rng.normal(size=d)
            e = e - (e @ k) / (k @ k) * k            # e perp k  =>  div(e sin(k.x)) = 0
            e = e / np.linalg.norm(e)
            ks.append(k); phis.append(rng.uniform(0, TWO_PI)); amps.append(amplitude * e)
    else:
        for c in range(d):
            for _ in range(per_component):
                k = _random_k(rng, d, kmax)
                e = np.zeros(d); e[c] = amplitude
                ks.append(k); phis.append(rng.uniform(0, TWO_PI)); amps.append(e)
    return SinusoidField(np.array(ks, float), np.array(phis, float), np.array(amps, float))


def _grid_points(n, device):
    """Node coordinates x_l = 2 pi l / n as a (d, N) tensor, x_1 fastest."""
    axes = [torch.arange(ni, dtype=torch.float64, device=device) * (TWO_PI / ni) for ni in n]
    mesh = torch.meshgrid(*reversed(axes), indexing="ij")
    return torch.stack([m.reshape(-1) for m in reversed(mesh)])


def _min_image(d):
    return torch.remainder(d + math.pi, TWO_PI) - math.pi


@dataclass
class Ellipsoid:
    centre: np.ndarray
    axes: np.ndarray
    rot: np.ndarray
    value: float


def _random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def _soft_ellipsoid(X, e: Ellipsoid, edge):
    """Smoothed indicator: 1/2 erfc(dist / (sqrt2 edge)), dist ~ (r-1)/|grad r| (analytic)."""
    c = torch.as_tensor(e.centre, dtype=X.dtype, device=X.device)[:, None]
    R = torch.as_tensor(e.rot, dtype=X.dtype, device=X.device)
    s = torch.as_tensor(e.axes, dtype=X.dtype, device=X.device)[:, None]
    u = (R.T @ _min_image(X - c)) / s
    r = torch.sqrt((u * u).sum(0)).clamp_min(1e-12)
    gr = torch.sqrt(((u / s) ** 2).sum(0)) / r
    dist = (r - 1.0) / gr.clamp_min(1e-12)
    return 0.5 * torch.special.erfc(dist / (math.sqrt(2.0) * edge))


@dataclass
class Phantom:
    kind: str
    params: list = field(default_factory=list)
    edge: float = 0.0
    lo: float = 0.0
    hi: float = 1.0

    def eval_raw(self, X):
        if self.kind == "gauss2d":
            out = torch.zeros(X.shape[1], dtype=X.dtype, device=X.device)
            for (cx, cy, sg, amp) in self.params:
                for ix in (-1, 0, 1):
                    for iy in (-1, 0, 1):
                        dx = X[0] - cx - ix * TWO_PI
                        dy = X[1] - cy - iy * TWO_PI
                        out = out + amp * torch.exp(-(dx * dx + dy * dy) / (2 * sg * sg))
            return out
        out = torch.zeros(X.shape[1], dtype=X.dtype, device=X.device)
        for e in self.params:
            out = out + e.value * _soft_ellipsoid(X, e, self.edge)
        return out

    def eval(self, X):
        return (self.eval_raw(X) - self.lo) / (self.hi - self.lo)


def _ellipsoid_set(rng, count, axis_lo, axis_hi):
    out = []
    for _ in range(count):
        centre = rng.uniform(0, TWO_PI, size=3)
        axes = rng.uniform(axis_lo, axis_hi, size=3)
        rot = _random_rotation(rng)
        value = rng.uniform(0.0, 1.0)
        out.append(Ellipsoid(centre, axes, rot, value))
    return out


def _shells(rng):
    """Brain-like phantom: 3 nested smoothed ellipsoid shells, 0.2/0.5/0.9 outside-in (R28)."""
    centre = np.pi + rng.uniform(-0.2, 0.2, size=3)
    outer = np.array([2.2, 2.6, 2.0]) * (1.0 + rng.uniform(-0.1, 0.1, size=3))
    rot = _random_rotation(rng)
    # nested indicators: 0.2*outer + 0.3*middle + 0.4*inner gives 0.2 / 0.5 / 0.9
    return [Ellipsoid(centre, outer, rot, 0.2), Ellipsoid(centre, 0.7 * outer, rot, 0.3),
            Ellipsoid(centre, 0.4 * outer, rot, 0.4)]


def _transport_exact(phantom, vstar, X1, continuity, nsub, chunk=1 << 22):
    """m1(x) = m0(Phi^{-1}(x)) [* exp(-int_0^1 div v*(X(t)) dt) for continuity].

    Backward characteristics X(1) = x, dX/dt = v*(X), integrated to t = 0 with
    classical RK4 and nsub substeps, in fp64, on the analytic v* (Liouville
    factor accumulated with the same RK4 stages).
    """
    out = torch.empty(X1.shape[1], dtype=X1.dtype, device=X1.device)
    dt = -1.0 / nsub
    for s0 in range(0, X1.shape[1], chunk):
        X = X1[:, s0:s0 + chunk].clone()
        logJ = torch.zeros(X.shape[1], dtype=X.dtype, device=X.device)
        for _ in range(nsub):
            k1, d1 = vstar.eval(X)
            k2, d2 = vstar.eval(X + 0.5 * dt * k1)
            k3, d3 = vstar.eval(X + 0.5 * dt * k2)
            k4, d4 = vstar.eval(X + dt * k3)
            X = X + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
            # d/dt log pi = -div v along the characteristic; integrating t: 1 -> 0
            logJ = logJ + dt / 6.0 * (d1 + 2 * d2 + 2 * d3 + d4)
        val = phantom.eval(torch.remainder(X, TWO_PI))
        if continuity:
            val = val * torch.exp(logJ)
        out[s0:s0 + chunk] = val
    return out


def _rescale_to_max_norm(vstar, X, target, chunk=1 << 22):
    """Scale v* so that max_x ||v*(x)||_2 over the grid equals target (R27)."""
    mx = 0.0
    for s0 in range(0, X.shape[1], chunk):
        v, _ = vstar.eval(X[:, s0:s0 + chunk])
        mx = max(mx, float(torch.sqrt((v * v).sum(0)).max()))
    vstar.scale = target / mx


def make_problem(config: int, n=None, device="cpu", nsub=32):
    """Build one seeded problem.  n overrides the grid (same recipe, smaller size).

    Returns dict with numpy fp64 arrays m0, m1 (numpy shape = reversed n),
    vstar (d, *shape), plus the solver settings of CONFIGS[config].
    """
    cfg = dict(CONFIGS[config])
    if n is not None:
        cfg["n"] = tuple(n)
    n = cfg["n"]
    d = len(n)
    rng = np.random.Generator(np.random.PCG64(SEED0 + config))
    X = _grid_points(n, device)
    shape = tuple(reversed(n))
    continuity = cfg["model"] == 1
    hmin = TWO_PI / max(n)

    if config == 1:
        params = [(rng.uniform(0, TWO_PI), rng.uniform(0, TWO_PI), rng.uniform(0.3, 0.6),
                   rng.uniform(0.5, 1.0)) for _ in range(4)]
        phantom = Phantom("gauss2d", params)
        # v* = 0.2 (sin x2 cos x1, -sin x1 cos x2) written as two sinusoid modes
        vstar = SinusoidField(np.array([[1.0, 1.0], [-1.0, 1.0]]), np.zeros(2),
                              np.array([[0.1, -0.1], [0.1, 0.1]]))
    elif config == 2:
        phantom = Phantom("ellipsoids", _ellipsoid_set(rng, 6, 0.3, 1.0), edge=1.0 * hmin)
        vstar = sample_sinusoid_field(rng, 3, 3, 3, 0.3)
    elif config == 3:
        phantom = Phantom("ellipsoids", _shells(rng), edge=1.0 * hmin)
        vstar = sample_sinusoid_field(rng, 3, 3, 4, 1.0, divfree=True)
        _rescale_to_max_norm(vstar, X, 0.3)
    elif config == 4:
        phantom = Phantom("ellipsoids", _shells(rng), edge=1.0 * hmin)
        vstar = sample_sinusoid_field(rng, 3, 4, 6, 1.0)
        _rescale_to_max_norm(vstar, X, 0.4)
    elif config == 5:
        phantom = Phantom("ellipsoids", _ellipsoid_set(rng, 32, 0.3, 1.0), edge=2.0 * hmin)
        vstar = sample_sinusoid_field(rng, 3, 8, 8, 1.0)
        _rescale_to_max_norm(vstar, X, 0.3)
    else:
        raise ValueError("config must be 1..5")

    m0 = phantom.eval(X)
    if config in (2, 5):  # affine normalisation to [0, 1] (R24); same map for m1
        phantom.lo, phantom.hi = float(m0.min()), float(m0.max())
        m0 = phantom.eval(X)
    m1 = _transport_exact(phantom, vstar, X, continuity, nsub)
    v, _ = vstar.eval(X)

    m0 = m0.cpu().numpy().reshape(shape)
    m1 = m1.cpu().numpy().reshape(shape)
    if config in (3, 4):  # independent N(0, 0.01^2) noise on m0 and m1 (R29)
        m0 = m0 + rng.normal(0.0, 0.01, size=shape)
        m1 = m1 + rng.normal(0.0, 0.01, size=shape)
    if config == 4:  # densities: clamp at 0, unit mass h^3 sum = 1 (R24, R29)
        vol = float(np.prod([TWO_PI / ni for ni in n]))
        m0 = np.maximum(m0, 0.0); m0 /= vol * m0.sum()
        m1 = np.maximum(m1, 0.0); m1 /= vol * m1.sum()
    cfg.update(config=config, m0=m0, m1=m1,
               vstar=v.cpu().numpy().reshape((d,) + shape))
    return cfg
