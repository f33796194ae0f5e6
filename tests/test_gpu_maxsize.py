"""Maximum size: BASELINE.json config 5 (512^3, advection, nt = 16, H2, alpha = 1e-3, w = 10)
on one GPU (workspace ~75 GB), at v = v*.  Sampled checks against the oracle, each operator
fed with the GPU's fp32 input to it (the whole fp64 oracle evaluation at 512^3 is far too
slow for a test): feet and forward steps at 4096 sampled nodes, the adjoint step with the
Heun factor (R7; div v from line derivatives) at 256 nodes, lam^S = m1 - m^S whole field,
the body force on sampled lines, g and s at sampled Fourier modes, dist."""
import numpy as np
import pytest
import torch

from gpu_common import rel_l2
from oracle import gradient as ogr
from oracle import spectral
from oracle.interp import interp_at, lagrange_weights
from oracle.spectral import Grid
from synth import make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-5
N = 512


def _line(field, a, i0, i1):
    """Line of `field` (numpy or torch, shape (N, N, N)) along paper axis a through (i0, i1)."""
    sl = [i0, i1]
    sl.insert(2 - a, slice(None))
    return field[tuple(sl)]


def _div_at(v, nodes):
    """div v at integer nodes (3, M) from spectral line derivatives (R3)."""
    out = np.zeros(nodes.shape[1])
    for q in range(nodes.shape[1]):
        x, y, z = nodes[:, q] % N
        out[q] = (spectral.deriv_line(v[0][z, y, :])[x] + spectral.deriv_line(v[1][z, :, x])[y]
                  + spectral.deriv_line(v[2][:, y, x])[z])
    return out


@pytest.fixture(scope="module")
def run():
    import paper_2510_08782_b200 as topt
    d = make_problem(5, device="cuda:0")
    assert tuple(d["n"]) == (N, N, N) and d["model"] == 0
    f32 = lambda x: np.asarray(x, dtype=np.float32)
    m0, m1, v = f32(d["m0"]), f32(d["m1"]), f32(d["vstar"])
    t = topt.Topt(topt.Config(n=(N, N, N), nt=d["nt"], model=0, reg_order=d["reg_order"], alpha=d["alpha"],
                              window=d["window"]), device="cuda:0")
    dv = lambda x: torch.tensor(x, device="cuda:0")
    g, s, sc = t.eval_gradient(dv(m0), dv(m1), dv(v))
    lam, b = t.adjoint()
    df, da = t.feet(dv(v))
    traj = t.forward(dv(m0), dv(v))
    torch.cuda.synchronize()
    out = dict(d=d, grid=Grid((N, N, N)), m0=m0, m1=m1, v=v.astype(np.float64), sc=t.scalars_dict(sc),
               g=g, s=s, lam=lam, b=b, df=df, da=da, traj=traj, t=t)
    yield out
    del out["t"]
    torch.cuda.empty_cache()


def _nodes(M, seed):
    return np.random.default_rng(seed).integers(0, N, size=(3, M))


def _at(tfield, nodes):
    """Values of a GPU field (N, N, N) at nodes (3, M) (paper order)."""
    idx = torch.tensor(nodes, device=tfield.device)
    return tfield[idx[2], idx[1], idx[0]].double().cpu().numpy()


def _ref_feet(run, nodes, sign):
    """dt I[v/h](l + sign dt/2 v_l/h) * sign (R6), at the nodes."""
    nt = run["d"]["nt"]
    dt, h = 1.0 / nt, 2 * np.pi / N
    vc = run["v"] / h
    vl = vc[:, nodes[2], nodes[1], nodes[0]]
    return np.stack([sign * dt * interp_at(vc[c], nodes, sign * 0.5 * dt * vl) for c in range(3)])


def test_feet(run):
    nodes = _nodes(4096, 1)
    for sign, key in ((-1.0, "df"), (1.0, "da")):
        ref = _ref_feet(run, nodes, sign)
        got = np.stack([_at(run[key][c], nodes) for c in range(3)])
        assert rel_l2(got, ref) < TOL, key


def test_forward_steps(run):
    nodes = _nodes(4096, 2)
    df = _ref_feet(run, nodes, -1.0)
    traj = run["traj"]
    for j in (0, run["d"]["nt"] - 1):
        mj = traj[j].double().cpu().numpy()
        ref = interp_at(mj, nodes, df)  # advection: no factor
        assert rel_l2(_at(traj[j + 1], nodes), ref) < TOL, j


def test_final_mismatch_and_adjoint_step(run):
    nt, lam, traj = run["d"]["nt"], run["lam"], run["traj"]
    mS = traj[nt].cpu().numpy()
    assert np.array_equal(lam[nt].cpu().numpy(), (run["m1"] - mS).astype(np.float32))
    nodes = _nodes(256, 3)
    da = _ref_feet(run, nodes, 1.0)
    dt = 1.0 / nt
    # Heun factor E_a = 1 + dt/2 (a' + b) + dt^2/2 a' b, a' = I[div v](Y), b = div v (R7)
    bdiv = _div_at(run["v"], nodes)
    ap = np.zeros(nodes.shape[1])
    for q in range(nodes.shape[1]):  # tricubic of div v at the foot from its 64 stencil nodes
        p = nodes[:, q] + da[:, q]
        ip = np.floor(p).astype(int)
        st = np.stack(np.meshgrid(*[np.arange(ip[a] - 1, ip[a] + 3) for a in range(3)], indexing="ij")).reshape(3, -1)
        vals = _div_at(run["v"], st)
        wx, wy, wz = (np.array(lagrange_weights(p[a] - ip[a])) for a in range(3))
        ap[q] = np.einsum("a,b,c,abc->", wx, wy, wz, vals.reshape(4, 4, 4))
    E = 1.0 + 0.5 * dt * (ap + bdiv) + 0.5 * dt * dt * ap * bdiv
    lam1 = lam[1].double().cpu().numpy()
    ref = interp_at(lam1, nodes, da) * E
    assert rel_l2(_at(lam[0], nodes), ref) < TOL


def test_body_force_sampled_lines(run):
    nt, lam, traj, b = run["d"]["nt"], run["lam"], run["traj"], run["b"]
    w = ogr.trapezoid_weights(nt)
    rng = np.random.default_rng(4)
    num = den = 0.0
    for a in range(3):
        for _ in range(8):
            i0, i1 = (int(x) for x in rng.integers(0, N, size=2))
            ref = np.zeros(N)
            for j in range(nt + 1):
                ref += w[j] * _line(lam[j], a, i0, i1).double().cpu().numpy() * \
                    spectral.deriv_line(_line(traj[j], a, i0, i1).double().cpu().numpy())  # (2.2)
            got = _line(b[a], a, i0, i1).double().cpu().numpy()
            num += np.sum((got - ref) ** 2)
            den += np.sum(ref ** 2)
    assert np.sqrt(num / den) < TOL


def test_gradient_preconditioner_modes_and_dist(run):
    grid, d = run["grid"], run["d"]
    alpha, p = d["alpha"], d["reg_order"]
    ks = [(0, 0, 0), (1, -2, 3), (6, 5, -4), (200, -17, 90)]
    gh, gref, sh, sref = [], [], [], []
    for k in ks:
        L = float(sum(x * x for x in k)) ** p
        Lt = L if L != 0.0 else 1.0
        coef = lambda fld, c: spectral.dft_coeff(grid, fld[c].double().cpu().numpy(), k)
        vh = np.array([spectral.dft_coeff(grid, run["v"][c], k) for c in range(3)])
        bh = np.array([coef(run["b"], c) for c in range(3)])
        g_k = np.array([coef(run["g"], c) for c in range(3)])
        s_k = np.array([coef(run["s"], c) for c in range(3)])
        gh.append(g_k); gref.append(alpha * L * vh + bh)
        sh.append(s_k); sref.append(-g_k / (alpha * Lt))
    gh, gref, sh, sref = map(np.array, (gh, gref, sh, sref))
    assert np.linalg.norm(gh - gref) / np.linalg.norm(gref) < TOL
    assert np.linalg.norm(sh - sref) / np.linalg.norm(sref) < TOL
    r = run["traj"][-1].double().cpu().numpy() - run["m1"]
    dist = 0.5 * spectral.inner(grid, r, r)
    assert abs(run["sc"]["dist"] - dist) <= TOL * dist
