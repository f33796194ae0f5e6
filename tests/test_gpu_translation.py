"""Exact translations through the GPU path (bitwise), the discrete form of the oracle pin "constant-v
advection on the periodic domain equals the exact translation" (tests/test_oracle_transport.py).

A constant velocity whose midpoint displacement dt/2 v/h is an integer k cells per axis (the fp32 v is
chosen so that the kernels' own product v * (dt/h) is exactly 2k): the midpoint interpolation then sits
on nodes (Lagrange weights exactly (0, 1, 0, 0), R5), both feet are exactly -2k / +2k cells, div v of a
constant field is exactly 0 (the line FFTs of a constant have exact zeros off the DC mode), so the Heun
factors are exactly 1, and every SL step is an exact periodic shift.  The feet, every forward slice and
every adjoint slice must therefore equal np.roll of the previous one BITWISE — on the tiled kernels
(3D, 64 x 32 x 32, displacements inside the halos and, with k = 2, beyond them: the L1 gathers) and on
the untiled 2D kernels."""
import numpy as np
import pytest

from gpu_common import case, dev, host, topt_for

pytestmark = pytest.mark.gpu


def _exact_velocity(d, k):
    """fp32 v_a per axis (numpy order: component a = x, y, z) with fp32(v_a * fp32(dt/h_a)) == 2 k_a."""
    n, nt = d["n"], d["nt"]
    dt = 1.0 / nt
    vel = []
    for a, ka in enumerate(k):
        gc = np.float32(dt / (2.0 * np.pi / n[a]))
        v = np.float32(2.0 * ka / float(gc))
        for _ in range(8):  # nudge by ulps until the kernels' fp32 product is exactly 2k
            p = np.float32(v * gc)
            if p == np.float32(2 * ka):
                break
            v = np.nextafter(v, np.float32(np.inf) if p < 2 * ka else np.float32(-np.inf), dtype=np.float32)
        assert np.float32(v * gc) == np.float32(2 * ka)
        vel.append(v)
    shape = d["m0"].shape
    return np.stack([np.full(shape, vv, dtype=np.float64) for vv in vel])


def _roll(f, shift_xyz):
    """np.roll of a [z][y][x] (or [y][x]) array by shift_xyz[a] along paper axis a."""
    nd = f.ndim
    return np.roll(f, tuple(shift_xyz[a] for a in range(nd)), axis=tuple(nd - 1 - a for a in range(nd)))


CASES = [
    (2, (64, 32, 32), (1, -1, 1)),   # tiled, feet 2 cells: shared-memory stencils
    (2, (64, 32, 32), (2, 0, -2)),   # feet 4 cells: beyond the 3-cell halo, L1 gathers
    (1, (64, 64), (1, -2)),          # 2D, untiled kernels
]


@pytest.mark.parametrize("cfg,n,k", CASES)
@pytest.mark.parametrize("model", [0, 1])
def test_translation_bitwise(cfg, n, k, model):
    d = case(cfg, n, model=model)
    v = _exact_velocity(d, k)
    t = topt_for(d)
    nd = len(n)
    df, da = t.feet(dev(v))
    df, da = host(df), host(da)
    for a in range(nd):
        assert np.all(df[a] == -2.0 * k[a]) and np.all(da[a] == 2.0 * k[a]), a
    traj = host(t.forward(dev(d["m0"]), dev(v)))
    assert np.array_equal(traj[0], d["m0"]) and np.any(traj[0] != _roll(traj[0], (1,) * nd))  # not trivial
    step = tuple(2 * ka for ka in k)
    for j in range(d["nt"]):
        assert np.array_equal(traj[j + 1], _roll(traj[j], step)), j
    t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(v))
    lam, _ = t.adjoint()
    lam = host(lam)
    assert np.array_equal(lam[d["nt"]], (d["m1"].astype(np.float32) - traj[d["nt"]].astype(np.float32)).astype(np.float64))
    assert np.any(lam[d["nt"]] != 0.0)
    back = tuple(-s for s in step)
    for j in range(d["nt"] - 1, -1, -1):
        assert np.array_equal(lam[j], _roll(lam[j + 1], back)), j
