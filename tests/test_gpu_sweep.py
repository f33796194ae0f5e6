"""Replica-sweep cells on the GPU (NEXT-3): a cell's row equals a direct solve of the same
setting, the paper's columns are consistent (dist, grad relative to v^0; converged => grad
<= eps; pde count = 2 per gradient evaluation + 1 per trial)."""
import pytest
import torch

import sweep

pytestmark = pytest.mark.gpu


def test_sweep_cells_on_gpu():
    cells = sweep.cells_for("wst", 64, 4, 1e-2, 5, 1, 2)[:2] + sweep.cells_for("alpha", 64, 4, 1e-2, 5, 1, 2)[:1]
    dev = torch.device("cuda:0")
    for c in cells:
        r = sweep.run_cell(c, "ngmres", 40, 5e-2, dev)
        assert 0.0 < r["dist"] <= 1.0
        assert r["grad"] > 0.0
        if r["converged"]:
            assert r["grad"] <= 5e-2
        assert r["iters"] >= 1 and r["pdes"] >= 2 * r["iters"]
        assert r["t_pdes"] <= r["tts"] and r["t_q"] + r["t_f"] <= r["t_pdes"] + 1e-6
        r2 = sweep.run_cell(c, "ngmres", 40, 5e-2, dev)  # deterministic GPU path
        assert (r2["iters"], r2["pdes"], r2["dist"], r2["grad"]) == (r["iters"], r["pdes"], r["dist"], r["grad"])
    print(sweep.format_table([r]))


def test_sweep_cell_matches_oracle_solve():
    """One alpha-grid cell (alpha = 5e-2, (sigma, tau) = (4, 2), w = 10) at 64^2 against the fp64
    oracle's GA-NGMRES solve of the same problem: the iteration count to eps = 5e-2 within +-1, the
    paper's dist and grad columns (relative to v^0) within 1e-3 (north_star tolerances)."""
    import numpy as np

    from gpu_common import case
    from oracle import gradient as ogr
    from oracle import solver as osolver
    cell = [c for c in sweep.cells_for("alpha", 64, 4, 0.0, 0, 0, 0)
            if (c["alpha"], c["sigma"], c["tau"], c["window"]) == (5e-2, 4, 2, 10)][0]
    r = sweep.run_cell(cell, "ngmres", 60, 5e-2, torch.device("cuda:0"))
    d = case(1, (64, 64), alpha=cell["alpha"], nt=cell["nt"])
    ref = osolver.solve(d["prob"], w=cell["window"], sigma=cell["sigma"], tau=cell["tau"], n_iter=60, eps_rel=5e-2)
    ref0 = ogr.evaluate(d["prob"], np.zeros_like(d["v"]))
    print(r["iters"], ref.iters, r["dist"], ref.info["dist"] / ref0["dist"], r["grad"], ref.grad_inf / ref.grad_inf0)
    assert ref.exit == osolver.CONVERGED and r["converged"]
    assert abs(r["iters"] - ref.iters) <= 1
    if r["iters"] == ref.iters:
        assert abs(r["dist"] - ref.info["dist"] / ref0["dist"]) <= 1e-3 * ref.info["dist"] / ref0["dist"]
        assert abs(r["grad"] - ref.grad_inf / ref.grad_inf0) <= 1e-3 * ref.grad_inf / ref.grad_inf0
