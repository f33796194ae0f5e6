"""Host logic of the replica sweep (sweep.py): the paper's grids (P:294,
P:505) and the round-robin deal of cells to ranks (every cell exactly once)."""
import sweep


def test_grids_match_the_paper():
    c = sweep.cells_for("wst", 128, 4, 1e-2, 20, 5, 1)
    assert len(c) == 7 * 4
    assert {(x["window"], x["sigma"], x["tau"]) for x in c} == {(w, s, t) for w in sweep.WST_W for s, t in sweep.WST_P}
    assert [x["alpha"] for x in sweep.cells_for("alpha", 128, 4, 1e-2, 20, 5, 1)] == [1e-1, 1e-2, 1e-3, 1e-4]
    assert [(x["n"], x["nt"]) for x in sweep.cells_for("mesh", 0, 0, 1e-2, 20, 5, 1)] == \
        [(64, 4), (128, 8), (256, 16), (512, 32)]


def test_cells_dealt_once():
    cells = sweep.cells_for("wst", 64, 4, 1e-2, 20, 5, 1)
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i, _ in sweep.cells_of_rank(cells, r, world))
        assert got == list(range(len(cells)))
