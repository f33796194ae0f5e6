"""GPU GA-NGMRES / GA-AA solves vs the fp64 oracle (BASELINE.json north_star):
after a fixed 20 iterations v and obj agree to relative 1e-3, and the iteration count to
the stopping tolerance agrees within +-1.  Also: tau = 0 invariance and
determinism of the GPU path (bitwise-identical reruns)."""
import numpy as np
import pytest
import torch

from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import solver as osolver

pytestmark = pytest.mark.gpu

CASES = [
    # (config recipe, grid, alpha override, w, sigma, tau)
    (1, (64, 64), None, 5, 1, 2),          # config 1: 2D, mixing period 3
    (2, (32, 32, 32), None, 5, 1, 0),      # config 2 recipe: H1, NGMRES(5)
    (3, (32, 32, 32), None, 5, 1, 1),      # config 3 recipe: incompressible, period 2
    # config 4 recipe (continuity), w = 3.  alpha = 1e-5 at 32^3 keeps all 20 iterations in the descent
    # regime; at 1e-4 the 32^3 problem reaches its fp64 noise floor after ~10 iterations (rel. grad
    # stalls at 7e-4, obj constant to 1e-8) where v is not determined by obj.
    (4, (32, 32, 32), 1e-5, 3, 1, 0),
]


def _oracle_solve(d, w, sigma, tau, n_iter, eps, method="ngmres", ordering="ga", replay=None):
    return osolver.solve(d["prob"], w=w, sigma=sigma, tau=tau, n_iter=n_iter, eps_rel=eps, method=method,
                         ordering=ordering, replay=replay)


def _gpu_solve(d, w, sigma, tau, n_iter, eps, method=0, ordering=0, replay=None):
    t = topt_for(d, window=w, sigma=sigma, tau=tau, max_iter=n_iter, eps_rel=eps, method=method,
                 ordering=ordering)
    if replay:
        t.set_step_replay(replay)
    v, rep = t.solve(dev(d["m0"]), dev(d["m1"]))
    return host(v), rep


@pytest.mark.parametrize("cfg,n,alpha,w,sigma,tau", CASES)
def test_twenty_iterations_match_oracle(cfg, n, alpha, w, sigma, tau):
    d = case(cfg, n, alpha=alpha)
    ref = _oracle_solve(d, w, sigma, tau, 20, 0.0)
    v, rep = _gpu_solve(d, w, sigma, tau, 20, 0.0)
    assert rep["iters"] == ref.iters == 20
    assert abs(rep["obj"] - ref.info["obj"]) <= 1e-3 * abs(ref.info["obj"])
    assert rel_l2(v, ref.v) <= 1e-3
    # replaying the oracle's step sequence removes Armijo branch flips
    v2, rep2 = _gpu_solve(d, w, sigma, tau, 20, 0.0, replay=ref.info["accepted"])
    assert rel_l2(v2, ref.v) <= 1e-3


@pytest.mark.parametrize("cfg,n,alpha,w,sigma,tau", CASES)
def test_iteration_count_to_tolerance(cfg, n, alpha, w, sigma, tau):
    d = case(cfg, n, alpha=alpha)
    ref = _oracle_solve(d, w, sigma, tau, 60, 5e-2)
    _, rep = _gpu_solve(d, w, sigma, tau, 60, 5e-2)
    assert ref.exit == osolver.CONVERGED
    assert rep["exit"] == 0
    assert abs(rep["iters"] - ref.iters) <= 1


@pytest.mark.parametrize("method,ordering", [(1, 0), (0, 1)])
def test_ga_aa_and_reverse_ordering_match_oracle(method, ordering):
    d = case(1, (64, 64))
    ref = _oracle_solve(d, 5, 2, 1, 12, 0.0, method="aa" if method else "ngmres",
                        ordering="a" if ordering else "ga")
    v, rep = _gpu_solve(d, 5, 2, 1, 12, 0.0, method=method, ordering=ordering,
                        replay=ref.info["accepted"])
    assert rep["iters"] == ref.iters
    assert rel_l2(v, ref.v) <= 1e-3


def test_tau_zero_any_sigma_identical_and_deterministic():
    d = case(1, (64, 64))
    va, _ = _gpu_solve(d, 3, 1, 0, 8, 0.0)
    vb, _ = _gpu_solve(d, 3, 4, 0, 8, 0.0)
    vc, _ = _gpu_solve(d, 3, 1, 0, 8, 0.0)
    assert np.array_equal(va, vb)
    assert np.array_equal(va, vc)


def test_python_solve_api():
    import paper_2510_08782_b200 as topt
    d = case(1, (64, 64))
    v, rep = topt.solve(torch.tensor(d["m0"], dtype=torch.float32), torch.tensor(d["m1"], dtype=torch.float32),
                        alpha=d["alpha"], nt=d["nt"], window=5, mixing_period=3, max_iter=40, device="cuda:0")
    assert rep["exit_name"] == "converged" and rep["iters"] < 40
