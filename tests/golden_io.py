"""Compact storage of oracle solve results for the native-grid solve-parity tests.

A 20-iteration fp64 oracle solve at 64^3 / 128^3 takes minutes to an hour of host time, too long
to repeat inside `pytest -m gpu`; `tools/make_solve_golden.py` (which calls only `oracle/` and
`synth/`) runs it once and stores the result here.  The final iterate v is smooth (it is a
combination of preconditioned steps s = -(alpha L~)^{-1} g), so it is stored as its Fourier
coefficients on the cube |k_i| <= K plus the l2 norm of the discarded tail; the parity test then
bounds ||v_gpu - v_ref||_2 RIGOROUSLY from above:

    ||v_g - v_r||^2 = ||P(v_g - v_r)||^2 + ||Q(v_g - v_r)||^2,   ||Q(v_g - v_r)|| <= ||Q v_g|| + ||Q v_r||

with P the projection on the stored cube and Q = I - P (Parseval, unnormalised DFT / n).
Storage encoding only: none of the method's arithmetic lives here.
"""
from __future__ import annotations

import numpy as np


def _cube_index(shape, K):
    """Index arrays selecting |k_i| <= K on the rfftn grid of `shape` (numpy order, last axis halved)."""
    idx = []
    for ax, n in enumerate(shape):
        if ax == len(shape) - 1:
            idx.append(np.arange(0, min(K, n // 2) + 1))
        else:
            kk = np.arange(n)
            kk = np.where(kk > n // 2, kk - n, kk)
            idx.append(np.nonzero(np.abs(kk) <= K)[0])
    return idx


def _parseval_weights(shape, sel_last):
    """rfft weights: interior modes of the halved axis count twice."""
    n = shape[-1]
    w = np.full(sel_last.shape, 2.0)
    w[sel_last == 0] = 1.0
    if n % 2 == 0:
        w[sel_last == n // 2] = 1.0
    return w


def _spec(v):
    """Per-component rfftn normalised so that sum |c|^2 (with rfft weights) = sum v^2."""
    shape = v.shape[1:]
    npts = int(np.prod(shape))
    return np.fft.rfftn(v, axes=tuple(range(1, v.ndim))) / np.sqrt(npts)


def _restrict(c, shape, K):
    idx = _cube_index(shape, K)
    return c[(slice(None),) + np.ix_(*idx)], idx


def _energy(c, shape, idx_last):
    w = _parseval_weights(shape, idx_last)
    return float(np.sum(w * np.abs(c) ** 2))


def encode_v(v, tail_rel=1e-4, kmax=None, prefix="v"):
    """Smallest cube K whose discarded tail is <= tail_rel ||v|| (or kmax); returns a dict."""
    v = np.asarray(v, dtype=np.float64)
    shape = v.shape[1:]
    c = _spec(v)
    tot = float(np.sum(v * v))
    kmax = kmax or max(shape) // 2
    for K in range(2, kmax + 1):
        cK, idx = _restrict(c, shape, K)
        tail2 = max(tot - _energy(cK, shape, idx[-1]), 0.0)
        if np.sqrt(tail2) <= tail_rel * np.sqrt(tot) or K == kmax:
            return {f"{prefix}_K": np.int64(K), f"{prefix}_coef": cK.astype(np.complex64),
                    f"{prefix}_tail": np.float64(np.sqrt(tail2)), f"{prefix}_norm": np.float64(np.sqrt(tot)),
                    f"{prefix}_shape": np.array(v.shape)}


def rel_l2_bound(v_gpu, g, prefix="v"):
    """Upper bound on ||v_gpu - v_ref|| / ||v_ref|| from the stored cube + tail (module docstring)."""
    v_gpu = np.asarray(v_gpu, dtype=np.float64)
    shape = v_gpu.shape[1:]
    assert tuple(v_gpu.shape) == tuple(g[f"{prefix}_shape"])
    K = int(g[f"{prefix}_K"])
    c = _spec(v_gpu)
    cK, idx = _restrict(c, shape, K)
    head = np.sqrt(_energy(cK - g[f"{prefix}_coef"].astype(np.complex128), shape, idx[-1]))
    tail_gpu = np.sqrt(max(float(np.sum(v_gpu * v_gpu)) - _energy(cK, shape, idx[-1]), 0.0))
    # complex64 storage rounding of the cube is ~6e-8 relative: negligible against 1e-3
    return float(np.sqrt(head ** 2 + (tail_gpu + float(g[f"{prefix}_tail"])) ** 2) / float(g[f"{prefix}_norm"]))
