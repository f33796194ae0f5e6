"""Periodic tricubic (bicubic in 2D) Lagrange interpolation.  TEST INFRASTRUCTURE ONLY.

The paper's semi-Lagrangian scheme evaluates fields off-grid but does
not name the interpolant.  Reading R5: tensor-product cubic
Lagrange on the 4 nodes i-1..i+2 per axis, taken modulo n (periodic), no
prefilter.  For position p (in cells) along an axis: i = floor(p), t = p - i,

    w_{-1} = -t (t-1)(t-2) / 6
    w_0    =  (t+1)(t-1)(t-2) / 2
    w_1    = -(t+1) t (t-2) / 2
    w_2    =  (t+1) t (t-1) / 6

Positions are always "node l plus displacement delta(l) in cells", which is
how every characteristic foot is expressed (reading R5; SURVEY §7 hard part 1).
Plain loops, one output point at a time (numba only compiles them).
"""
from __future__ import annotations

import math

import numba
import numpy as np


@numba.njit(cache=True, inline="always")
def lagrange_weights(t):
    wm1 = -t * (t - 1.0) * (t - 2.0) / 6.0
    w0 = (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0
    w1 = -(t + 1.0) * t * (t - 2.0) / 2.0
    w2 = (t + 1.0) * t * (t - 1.0) / 6.0
    return wm1, w0, w1, w2


@numba.njit(parallel=True, cache=True)
def _interp3(f, dx, dy, dz):
    nz, ny, nx = f.shape
    out = np.empty_like(f)
    for k in numba.prange(nz):
        for j in range(ny):
            for i in range(nx):
                px = i + dx[k, j, i]
                py = j + dy[k, j, i]
                pz = k + dz[k, j, i]
                ix = math.floor(px)
                iy = math.floor(py)
                iz = math.floor(pz)
                wx = lagrange_weights(px - ix)
                wy = lagrange_weights(py - iy)
                wz = lagrange_weights(pz - iz)
                acc = 0.0
                for c in range(4):
                    zz = (iz - 1 + c) % nz
                    for b in range(4):
                        yy = (iy - 1 + b) % ny
                        for a in range(4):
                            xx = (ix - 1 + a) % nx
                            acc += wz[c] * wy[b] * wx[a] * f[zz, yy, xx]
                out[k, j, i] = acc
    return out


@numba.njit(parallel=True, cache=True)
def _interp2(f, dx, dy):
    ny, nx = f.shape
    out = np.empty_like(f)
    for j in numba.prange(ny):
        for i in range(nx):
            px = i + dx[j, i]
            py = j + dy[j, i]
            ix = math.floor(px)
            iy = math.floor(py)
            wx = lagrange_weights(px - ix)
            wy = lagrange_weights(py - iy)
            acc = 0.0
            for b in range(4):
                yy = (iy - 1 + b) % ny
                for a in range(4):
                    xx = (ix - 1 + a) % nx
                    acc += wy[b] * wx[a] * f[yy, xx]
            out[j, i] = acc
    return out


@numba.njit(parallel=True, cache=True)
def _interp3_at(f, px, py, pz):
    nz, ny, nx = f.shape
    out = np.empty(px.shape[0])
    for q in numba.prange(px.shape[0]):
        ix = math.floor(px[q])
        iy = math.floor(py[q])
        iz = math.floor(pz[q])
        wx = lagrange_weights(px[q] - ix)
        wy = lagrange_weights(py[q] - iy)
        wz = lagrange_weights(pz[q] - iz)
        acc = 0.0
        for c in range(4):
            zz = (iz - 1 + c) % nz
            for b in range(4):
                yy = (iy - 1 + b) % ny
                for a in range(4):
                    xx = (ix - 1 + a) % nx
                    acc += wz[c] * wy[b] * wx[a] * f[zz, yy, xx]
        out[q] = acc
    return out


def interp_at(f, nodes, delta):
    """I[f](l + delta) at a list of nodes only (3D): nodes int (3, M) in paper order
    (x_1 index first), delta (3, M) displacements in cells.  The same formula as `interp`
    one point at a time; used to check full-size fields at sampled points."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    pos = np.asarray(nodes, dtype=np.float64) + np.asarray(delta, dtype=np.float64)
    return _interp3_at(f, np.ascontiguousarray(pos[0]), np.ascontiguousarray(pos[1]), np.ascontiguousarray(pos[2]))


def interp(f, delta):
    """I[f](l + delta(l)) for every node l.

    f: scalar field, numpy shape (n_d, ..., n_1), fp64.
    delta: displacement in cells, shape (d, *f.shape); delta[a] along paper axis a.
    """
    f = np.ascontiguousarray(f, dtype=np.float64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    if f.ndim == 3:
        return _interp3(f, delta[0], delta[1], delta[2])
    if f.ndim == 2:
        return _interp2(f, delta[0], delta[1])
    raise ValueError("interp supports d = 2 or 3")


def interp_vec(u, delta):
    """Componentwise interpolation of a vector field u (shape (d, *shape))."""
    return np.stack([interp(u[c], delta) for c in range(u.shape[0])])
