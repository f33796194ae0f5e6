"""z-slab decomposition: P slabs emulated on one GPU — halo exchange, z<->y
all-to-all transposes and all-reduces become device copies — must reproduce the single-slab
evaluation (the same kernels on the same data; only summation order and the FFT z passes'
tiling differ) and the oracle.  The NCCL transport moves the same bytes between processes."""
import numpy as np
import pytest

from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr
from oracle import spectral

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("model", [0, 1, 2])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_eval_gradient_slab_invariance(model, P, transport):
    """transport "nccl": the emulated pack / send-recv / unpack copies; "p2p": the pull kernel
    reading every chunk straight from the owning slab (the kernel of the CUDA-IPC transport)."""
    d = case(2, (64, 32, 32), model=model)
    if model == 2:
        d["v"] = spectral.leray(d["grid"], d["v"]).astype(np.float32).astype(np.float64)
    t1 = topt_for(d)
    g1, s1, sc1 = t1.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    tp = topt_for(d, world=P)
    tp.set_transport(transport)
    gp, sp, scp = tp.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    g1, s1, gp, sp = host(g1), host(s1), host(gp), host(sp)
    assert rel_l2(gp, g1) < 1e-6
    assert rel_l2(sp, s1) < 1e-6
    a, b = t1.scalars_dict(sc1), tp.scalars_dict(scp)
    for k in ("obj", "dist", "reg", "grad_inf", "gs", "slv", "sls"):
        assert abs(a[k] - b[k]) <= 1e-6 * abs(a[k]) + 1e-30, k
    ref = ogr.evaluate(d["prob"], d["v"])
    assert rel_l2(gp, ref["g"]) < 1e-5
    assert rel_l2(sp, ref["s"]) < 1e-5


def test_objective_slab_invariance():
    d = case(2, (64, 32, 32))
    o1 = topt_for(d).objective(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    o4 = topt_for(d, world=4).objective(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    for k in ("obj", "dist", "reg"):
        assert abs(o1[k] - o4[k]) <= 1e-6 * abs(o1[k]), k


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("P", [2, 8])
def test_solve_slab_invariance(P, transport):
    """12 GA-NGMRES iterations on P emulated slabs vs one slab."""
    d = case(2, (64, 32, 32))
    t1 = topt_for(d, max_iter=12, eps_rel=0.0)
    v1, r1 = t1.solve(dev(d["m0"]), dev(d["m1"]))
    tp = topt_for(d, world=P, max_iter=12, eps_rel=0.0)
    tp.set_transport(transport)
    vp, rp = tp.solve(dev(d["m0"]), dev(d["m1"]))
    assert rp["iters"] == r1["iters"] == 12
    assert abs(rp["obj"] - r1["obj"]) <= 1e-5 * abs(r1["obj"])
    assert rel_l2(host(vp), host(v1)) < 1e-4


@pytest.mark.parametrize("P", [2, 4])
def test_p2p_pull_equals_copy_transport_bitwise(P):
    """Both transports move the same bytes: the evaluation and a short solve agree bitwise."""
    d = case(2, (64, 32, 32), model=1)
    out = {}
    for tr in ("nccl", "p2p"):
        t = topt_for(d, world=P, max_iter=3, eps_rel=0.0)
        t.set_transport(tr)
        g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
        v, rep = t.solve(dev(d["m0"]), dev(d["m1"]))
        out[tr] = (host(g), host(s), host(v), rep["obj"])
    for a, b in zip(out["nccl"][:3], out["p2p"][:3]):
        assert np.array_equal(a, b)
    assert out["nccl"][3] == out["p2p"][3]


def test_transport_and_peer_arguments_checked():
    import ctypes

    import paper_2510_08782_b200 as topt
    LIB = topt._lib.LIB
    d = case(2, (32, 32, 32))
    t = topt_for(d, world=2)
    assert LIB.topt_set_transport(t.ctx, 5) != 0
    bases = (ctypes.c_void_p * 3)()
    assert LIB.topt_set_peer_workspaces(t.ctx, bases, 3) != 0   # count != world
    assert LIB.topt_set_peer_workspaces(t.ctx, bases, 0) == 0   # clear


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("scale", [4.0, 24.0])
def test_large_feet_window_matches_single_slab(P, scale):
    """Feet far beyond the stored 4-plane halo (|delta_z| ~ 5 and ~ 28 cells on a 32-plane grid:
    the window is sized from max |delta_z|, gathered over several slabs when it is wider than
    one (P = 8: 4 planes per slab), and wraps a whole period at the larger scale; SL has no CFL
    limit): the P-slab evaluation equals the single-slab one."""
    d = case(2, (64, 32, 32), model=1, scale=scale)
    t1 = topt_for(d)
    df, _ = t1.feet(dev(d["v"]))
    dz = float(np.max(np.abs(host(df)[2])))
    assert dz > 3.0 and (scale < 10 or dz > 16.0), dz
    g1, s1, sc1 = t1.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    tp = topt_for(d, world=P)
    gp, sp, scp = tp.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    assert rel_l2(host(gp), host(g1)) < 1e-6
    assert rel_l2(host(sp), host(s1)) < 1e-6
    a, b = t1.scalars_dict(sc1), tp.scalars_dict(scp)
    for k in ("obj", "dist", "grad_inf", "gs"):
        assert abs(a[k] - b[k]) <= 1e-6 * abs(a[k]), k


@pytest.mark.parametrize("P", [2, 4])
def test_solve_with_trial_feet_beyond_halo(P):
    """GA-NGMRES from v^0 = 4 v*: the Armijo trials' feet reach |delta_z| > 3 cells.  No trial is
    rejected for halo reasons (the window is sized per evaluation), so the P-slab solve takes the
    single-slab step sequence."""
    d = case(2, (64, 32, 32), scale=4.0)
    t1 = topt_for(d)
    df, _ = t1.feet(dev(d["v"]))
    assert float(np.max(np.abs(host(df)[2]))) > 3.0
    t1 = topt_for(d, max_iter=8, eps_rel=0.0)
    v1, r1 = t1.solve(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    tp = topt_for(d, world=P, max_iter=8, eps_rel=0.0)
    vp, rp = tp.solve(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    assert rp["iters"] == r1["iters"] == 8
    assert (rp["obj_evals"], rp["grad_evals"], rp["rho"]) == (r1["obj_evals"], r1["grad_evals"], r1["rho"])
    assert abs(rp["obj"] - r1["obj"]) <= 1e-6 * abs(r1["obj"])
    assert rel_l2(host(vp), host(v1)) < 1e-5


def test_bench_slab_check_on_emulated_slabs():
    """bench.py's one-time z-slab check at N > 1 (_slab_check + slab_agreement), run here on an
    emulated 4-slab context (all slabs in one process: rank 0 of a world of 1 owns the whole grid):
    the z-slab and whole-grid evaluations must agree, and a g off by 1e-3 must fail the check."""
    import torch

    import bench
    import paper_2510_08782_b200 as topt
    from synth import make_problem
    d = make_problem(2, (64, 32, 32))
    cfgp = dict(n=tuple(d["n"]), nt=d["nt"], model=d["model"], reg_order=d["reg_order"], alpha=d["alpha"])
    tp = topt.Topt(topt.Config(window=d["window"], **cfgp), device="cuda:0", world=4)
    local = bench._slab_check(tp, topt, d, cfgp, torch.device("cuda:0"), 0, 1, d["m0"], d["m1"], d["vstar"])
    res = bench.slab_agreement(local, 1)
    assert res["ok"] and res["g_rel_l2"] < 1e-6, res
    assert local["graphs_diff"] == 0.0  # segmented graph replay == eager, bitwise
    assert not bench.slab_agreement(dict(local, dl=local["rl"] * 1e-6), 1)["ok"]


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_slab_graphs_equal_eager_bitwise(P, transport):
    """z-slab evaluations replay CUDA graphs captured in three segments between the host's two
    window decisions: bitwise the eager evaluation on first capture, on replay,
    and when a new v changes the decisions (feet beyond the 4-plane halo: the window path, a new
    segment captured while the earlier ones are replayed) and changes them back."""
    import torch
    d = case(2, (64, 32, 32), model=1)
    wide = case(2, (64, 32, 32), model=1, scale=4.0)
    vs = [dev(d["v"]), dev(d["v"]), dev(wide["v"]), dev(d["v"]), dev(wide["v"])]
    m0, m1 = dev(d["m0"]), dev(d["m1"])
    res = {}
    for graphs in (False, True):
        t = topt_for(d, world=P)
        t.set_transport(transport)
        t.set_graphs(graphs)
        g = torch.empty_like(vs[0])
        s = torch.empty_like(vs[0])
        sc = torch.zeros(16, dtype=torch.float64, device=vs[0].device)
        v = torch.empty_like(vs[0])  # one pointer key: the decisions alone pick the segments
        out = []
        for vk in vs:
            v.copy_(vk)
            l0 = t.launch_count()
            t.eval_gradient(m0, m1, v, g, s, sc)
            torch.cuda.synchronize()
            out.append((host(g).copy(), host(s).copy(), host(sc).copy(), t.launch_count() - l0))
        res[graphs] = out
    for k, (a, b) in enumerate(zip(res[False], res[True])):
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y), k
        assert a[3] == b[3] > 0, k  # replayed graphs count the kernels they contain
    assert not np.array_equal(res[True][1][0], res[True][2][0])  # the wide v really differs


def test_slab_graphs_follow_the_transport():
    """Captured z-slab segments bake the transport in: switching it drops them, so the replayed
    evaluation launches the new transport's kernels (the same count as the eager path)."""
    import torch
    d = case(2, (64, 32, 32), model=1)
    m0, m1, v = dev(d["m0"]), dev(d["m1"]), dev(d["v"])

    def launches(t):
        g = torch.empty_like(v)
        s = torch.empty_like(v)
        sc = torch.zeros(16, dtype=torch.float64, device=v.device)
        n = []
        for _ in range(2):
            l0 = t.launch_count()
            t.eval_gradient(m0, m1, v, g, s, sc)
            torch.cuda.synchronize()
            n.append(t.launch_count() - l0)
        return n

    eager = {}
    for tr in ("nccl", "p2p"):
        t = topt_for(d, world=4)
        t.set_transport(tr)
        t.set_graphs(False)
        eager[tr] = launches(t)[0]
    assert eager["nccl"] != eager["p2p"]
    t = topt_for(d, world=4)
    for tr in ("nccl", "p2p", "nccl"):
        t.set_transport(tr)
        assert launches(t) == [eager[tr]] * 2, tr
