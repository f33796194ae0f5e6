"""Line search, fixed-point map and the NGMRES / AA family (fp64).  TEST INFRASTRUCTURE ONLY.

PAPER.md anchors:
  (2.3)/(2.4) line search v + rho s, Armijo obj(v+rho s) < obj(v) + rho c <g,s>,
              c = 1e-4, start at 1, halve; keep rho in memory, double it when the
              first trial passes
  (2.7)       q(v) = v - rho (alpha L)^{-1} g(v); r(v) = v - q(v)
  Alg. 1      NGMRES(w)
  Alg. 2      AA(w)
  Alg. 3      GA-NGMRES(w; sigma, tau): FP when mod(k, sigma+tau) >= sigma
  aNGMRES(w)[sigma]-FP[tau] reverse ordering (switch mod(k,sigma+tau) < tau)

Readings:
  R12 no cap on rho; 50 halvings without acceptance => STAGNATED; one rho state
      per solve shared by FP and NGMRES steps
  R13 w_k = min(k, w) and the LSQ has w_k + 1 columns i = 0..w_k
  R15 LSQ: minimum-norm solution, singular values below 1e-6 sigma_max dropped
      (fp64 SVD of the column matrix); all-zero columns => beta = 0 (R26)
  R16 iterations count completed updates; stop when
      ||g(v^{k+1})||_inf <= eps ||g(v^0)||_inf or k+1 >= n_iter
  R17 FP steps reuse g(q) as g(v^{k+1}); NGMRES steps evaluate g(v^{k+1}) anew
  R19 v^0 = 0; R21 the stop test uses the raw gradient
  R9  incompressible: the mixed iterate is re-projected with P_L
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import gradient as _gradient
from . import spectral

CONVERGED, ITER_CAP, STAGNATED = 0, 1, 2


def lsq_min_norm(cols, rhs, rcond=1e-6):
    """argmin_beta || rhs + sum_i beta_i cols_i ||_2, minimum-norm, truncated SVD (R15)."""
    if len(cols) == 0:
        return np.zeros(0)
    C = np.stack([c.ravel() for c in cols], axis=1)
    U, sv, Vt = np.linalg.svd(C, full_matrices=False)
    if sv.size == 0 or sv[0] == 0.0:
        return np.zeros(len(cols))
    keep = sv > rcond * sv[0]
    coef = (U[:, keep].T @ (-rhs.ravel())) / sv[keep]
    return Vt[keep].T @ coef


@dataclass
class LineSearchState:
    rho: float = 1.0
    c: float = 1e-4
    max_backtracks: int = 50
    trials: int = 0
    stagnated: bool = False
    replay: list = field(default_factory=list)  # optional forced rho sequence (debug)
    accepted: list = field(default_factory=list)  # accepted rho per q evaluation (for replay)


class TransportFP:
    """The RPGD fixed-point map q of (2.7) for a transport Problem."""

    def __init__(self, prob: _gradient.Problem):
        self.prob = prob
        self.grad_evals = 0
        self.obj_evals = 0

    def gradient(self, v):
        self.grad_evals += 1
        return _gradient.evaluate(self.prob, v)

    def objective(self, v):
        self.obj_evals += 1
        return _gradient.objective(self.prob, v)["obj"]

    def project(self, v):
        if self.prob.model == _gradient.INCOMPRESSIBLE:
            return spectral.leray(self.prob.grid, v)
        return v

    def q(self, v, info, ls: LineSearchState):
        """Armijo backtracking with memory along s = -(alpha L~)^{-1} g."""
        s, obj0, gs = info["s"], info["obj"], info["gs"]
        if ls.replay:
            rho = ls.replay.pop(0)
            ls.rho = rho
            ls.accepted.append(rho)
            return v + rho * s
        rho = ls.rho
        for t in range(ls.max_backtracks + 1):
            vt = v + rho * s
            ls.trials += 1
            if self.objective(vt) < obj0 + rho * ls.c * gs:
                ls.rho = 2.0 * rho if t == 0 else rho
                ls.accepted.append(rho)
                return vt
            rho *= 0.5
        ls.stagnated = True
        return v

    def pde_solves(self):
        return 2 * self.grad_evals + self.obj_evals


class LinearRichardsonFP:
    """q(v) = v - omega (A v - b), g(v) = A v - b: the linear setting of P:211 / P:294."""

    def __init__(self, A, b, omega):
        self.A, self.b, self.omega = A, b, omega
        self.grad_evals = 0
        self.obj_evals = 0

    def gradient(self, v):
        self.grad_evals += 1
        return {"g": self.A @ v - self.b}

    def project(self, v):
        return v

    def q(self, v, info, ls):
        return v - self.omega * info["g"]


@dataclass
class SolveResult:
    v: np.ndarray
    iters: int
    exit: int
    grad_inf0: float
    grad_inf: float
    rel_grad: list
    iterates: list
    betas: list
    info: dict


def ga_ngmres(fp, v0, w, sigma=1, tau=0, n_iter=200, eps_rel=5e-2, ordering="ga",
              ls: LineSearchState | None = None, keep_iterates=False):
    """GA-NGMRES(w; sigma, tau), Alg. 3; tau = 0 gives NGMRES(w), Alg. 1.

    ordering = "ga": FP when mod(k, sigma+tau) >= sigma (Alg. 3 line 5);
    ordering = "a" : aNGMRES(w)[sigma]-FP[tau], FP when mod(k, sigma+tau) < tau.
    """
    if sigma < 1 or tau < 0 or w < 0:
        raise ValueError("need sigma >= 1, tau >= 0, w >= 0")
    ls = ls or LineSearchState()
    v = np.array(v0, dtype=np.float64)
    info = fp.gradient(v)
    g0 = float(np.max(np.abs(info["g"])))
    hist = deque([(v, info["g"])], maxlen=w + 1)  # most recent last
    rel, iterates, betas = [], [v] if keep_iterates else [], []
    k, exit_code = 0, ITER_CAP
    while True:
        qv = fp.q(v, info, ls)
        if ls.stagnated:
            exit_code = STAGNATED
            break
        info_q = fp.gradient(qv)
        period = sigma + tau
        fp_step = (k % period >= sigma) if ordering == "ga" else (k % period < tau)
        if fp_step:
            v_new, info_new = qv, info_q
        else:
            gq = info_q["g"]
            past = list(reversed(hist))  # i = 0..w_k : v^{k-i}
            beta = lsq_min_norm([gq - gi for (_, gi) in past], gq)
            betas.append(beta)
            v_new = qv.copy()
            for bi, (vi, _) in zip(beta, past):
                v_new += bi * (qv - vi)
            v_new = fp.project(v_new)
            info_new = fp.gradient(v_new)
        v, info = v_new, info_new
        hist.append((v, info["g"]))
        k += 1
        gi = float(np.max(np.abs(info["g"])))
        rel.append(gi / g0 if g0 > 0 else 0.0)
        if keep_iterates:
            iterates.append(v)
        if gi <= eps_rel * g0:
            exit_code = CONVERGED
            break
        if k >= n_iter:
            exit_code = ITER_CAP
            break
    return SolveResult(v, k, exit_code, g0, float(np.max(np.abs(info["g"]))), rel, iterates,
                       betas, info)


def ga_aa(fp, v0, w, sigma=1, tau=0, n_iter=200, eps_rel=5e-2, ordering="ga",
          ls: LineSearchState | None = None, keep_iterates=False):
    """GA-AA(w; sigma, tau): Alg. 2 under the Alg. 3 schedule.

    AA step: r_k = v^k - q(v^k); xi = argmin ||r_k + sum_{i=1}^{w_k} xi_i (r_k - r_{k-i})||;
    v^{k+1} = q(v^k) + sum_{i=1}^{w_k} xi_i (q(v^k) - q(v^{k-i})).
    """
    ls = ls or LineSearchState()
    v = np.array(v0, dtype=np.float64)
    info = fp.gradient(v)
    g0 = float(np.max(np.abs(info["g"])))
    hist = deque(maxlen=w + 1)  # (r_i, q_i), most recent last
    rel, iterates, betas = [], [v] if keep_iterates else [], []
    k, exit_code = 0, ITER_CAP
    while True:
        qv = fp.q(v, info, ls)
        if ls.stagnated:
            exit_code = STAGNATED
            break
        r = v - qv
        period = sigma + tau
        fp_step = (k % period >= sigma) if ordering == "ga" else (k % period < tau)
        past = list(reversed(hist))[: min(k, w)]  # i = 1..w_k
        if fp_step or not past:
            v_new = qv
        else:
            xi = lsq_min_norm([r - ri for (ri, _) in past], r)
            betas.append(xi)
            v_new = qv.copy()
            for xj, (_, qj) in zip(xi, past):
                v_new += xj * (qv - qj)
            v_new = fp.project(v_new)
        hist.append((r, qv))
        info = fp.gradient(v_new)
        v = v_new
        k += 1
        gi = float(np.max(np.abs(info["g"])))
        rel.append(gi / g0 if g0 > 0 else 0.0)
        if keep_iterates:
            iterates.append(v)
        if gi <= eps_rel * g0:
            exit_code = CONVERGED
            break
        if k >= n_iter:
            exit_code = ITER_CAP
            break
    return SolveResult(v, k, exit_code, g0, float(np.max(np.abs(info["g"]))), rel, iterates,
                       betas, info)


def solve(prob: _gradient.Problem, w, sigma=1, tau=0, n_iter=200, eps_rel=5e-2,
          method="ngmres", ordering="ga", replay=None):
    """Convenience: GA-NGMRES (or GA-AA) on a transport problem from v^0 = 0."""
    fp = TransportFP(prob)
    ls = LineSearchState(replay=list(replay) if replay else [])
    v0 = np.zeros((prob.grid.d,) + prob.grid.shape)
    run = ga_ngmres if method == "ngmres" else ga_aa
    res = run(fp, v0, w, sigma, tau, n_iter, eps_rel, ordering, ls)
    res.info = dict(res.info)
    res.info.update(grad_evals=fp.grad_evals, obj_evals=fp.obj_evals,
                    pde_solves=fp.pde_solves(), rho=ls.rho, trials=ls.trials,
                    accepted=list(ls.accepted))
    return res
