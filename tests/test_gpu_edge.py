"""Edge and degenerate cases of the GPU path against the oracle (north_star tolerances):
identical images at v = 0 (lam = 0, so b = g = s = 0 exactly, and the line search can only
stagnate, R12), the smallest supported grids (one radix-8 line per axis, a single SL tile),
a single time step (trapezoid weights 1/2, 1/2), and the H1 / H3 regularisers (R4)."""
import numpy as np
import pytest

from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr
from oracle import solver as osolver

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("model", [0, 1, 2])
def test_identical_images_zero_velocity(model):
    d = case(2, (32, 32, 32), model=model)
    t = topt_for(d, max_iter=5, eps_rel=1e-3)
    z = np.zeros_like(d["v"])
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m0"]), dev(z))
    assert np.all(host(g) == 0.0) and np.all(host(s) == 0.0)
    sd = t.scalars_dict(sc)
    assert sd["obj"] == 0.0 and sd["grad_inf"] == 0.0
    v, rep = t.solve(dev(d["m0"]), dev(d["m0"]))
    assert np.all(host(v) == 0.0)
    d["prob"].m1 = d["prob"].m0
    ref = osolver.solve(d["prob"], w=5, n_iter=5, eps_rel=1e-3)
    assert rep["exit"] == ref.exit == osolver.STAGNATED


@pytest.mark.parametrize("cfg,n", [(2, (8, 8, 8)), (1, (8, 8)), (2, (32, 8, 8))])
@pytest.mark.parametrize("model", [0, 1])
def test_smallest_grids(cfg, n, model):
    d = case(cfg, n, model=model, scale=0.25)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    ref = ogr.evaluate(d["prob"], d["v"])
    assert rel_l2(host(g), ref["g"]) < TOL
    assert rel_l2(host(s), ref["s"]) < TOL
    assert abs(t.scalars_dict(sc)["obj"] - ref["obj"]) <= TOL * abs(ref["obj"])


@pytest.mark.parametrize("nt", [1, 2])
def test_few_time_steps(nt):
    d = case(2, (32, 32, 32), nt=nt, model=1)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    ref = ogr.evaluate(d["prob"], d["v"])
    assert rel_l2(host(g), ref["g"]) < TOL
    assert abs(t.scalars_dict(sc)["obj"] - ref["obj"]) <= TOL * abs(ref["obj"])


@pytest.mark.parametrize("p", [1, 3])
@pytest.mark.parametrize("model", [0, 2])
def test_h1_h3_regularisers(p, model):
    d = case(2, (32, 32, 32), model=model, reg_order=p)
    if model == 2:
        from oracle import spectral
        d["v"] = spectral.leray(d["grid"], d["v"]).astype(np.float32).astype(np.float64)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    ref = ogr.evaluate(d["prob"], d["v"])
    assert rel_l2(host(g), ref["g"]) < TOL
    assert rel_l2(host(s), ref["s"]) < TOL
    sd = t.scalars_dict(sc)
    assert abs(sd["reg"] - ref["reg"]) <= TOL * abs(ref["reg"])
