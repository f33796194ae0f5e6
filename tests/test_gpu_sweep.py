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
