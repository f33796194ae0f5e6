"""The NGMRES machinery of the GPU solver (fp64 Gram multi-dot, host fp64 LSQ, mixing kernel) on a
LINEAR fixed-point map, against the fp64 oracle's NGMRES on the same map:
q(v) = v - omega (A v - b), A = I + alpha L applied spectrally (R4).  In the linear case
NGMRES(infinity) produces the GMRES iterates, pinned in the oracle by
tests/test_oracle_solver.py; here the GPU iterates must follow the oracle's, and their residuals
must be non-increasing (GMRES minimises the residual over a growing Krylov space)."""
import numpy as np
import pytest

from gpu_common import dev, host, rel_l2, topt_for
from oracle import solver as osolver
from oracle import spectral
from oracle.spectral import Grid

pytestmark = pytest.mark.gpu


class _SpectralA:
    """A = I + alpha L (oracle fp64), usable as `A @ v` by oracle.solver.LinearRichardsonFP."""

    def __init__(self, grid, alpha, p):
        self.grid, self.alpha, self.p = grid, alpha, p

    def __matmul__(self, v):
        return v + self.alpha * spectral.apply_L(self.grid, v, self.p)


def _problem(n, alpha, p, seed):
    grid = Grid(n)
    rng = np.random.default_rng(seed)
    b = np.stack([spectral.gaussian_blur(grid, rng.normal(size=grid.shape), 1.5) for _ in range(len(n))])
    b = b.astype(np.float32).astype(np.float64)
    kmax2 = sum((x // 2) ** 2 for x in n)
    omega = 1.0 / (1.0 + alpha * kmax2 ** p)  # Richardson step below 2 / lambda_max
    return grid, b, omega


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


class _Fp32StorageFP(osolver.LinearRichardsonFP):
    """The oracle's map and NGMRES with every vector the GPU path STORES rounded to fp32 (q, g and the
    mixed iterate, through the q / gradient / project hooks of oracle.solver.ga_ngmres); arithmetic
    stays fp64.  Its distance from the fp64 oracle is what fp32 storage alone costs this method."""

    def gradient(self, v):
        return {"g": _f32(super().gradient(v)["g"])}

    def q(self, v, info, ls):
        return _f32(super().q(v, info, ls))

    def project(self, v):
        return _f32(v)


@pytest.mark.parametrize("n,alpha,p,w,iters", [((16, 16, 16), 1e-2, 2, 30, 12), ((32, 32), 1e-3, 2, 30, 12),
                                               ((16, 16, 16), 1e-2, 1, 3, 10)])
def test_linear_ngmres_matches_oracle(n, alpha, p, w, iters):
    grid, b, omega = _problem(n, alpha, p, 2510)
    d = dict(n=n, nt=1, model=0, reg_order=p, alpha=alpha)
    t = topt_for(d, window=w)
    v, res = t.linear_ngmres(dev(b), omega, iters)
    fp = osolver.LinearRichardsonFP(_SpectralA(grid, alpha, p), b, omega)
    ref = osolver.ga_ngmres(fp, np.zeros_like(b), w, n_iter=iters, eps_rel=0.0, keep_iterates=True)
    ref_res = [float(np.linalg.norm(fp.A @ x - b)) for x in ref.iterates]
    assert ref.iters == iters
    # fp32 storage alone moves GMRES iterates on A = I + alpha L (large early beta, e.g. 236, 68, 33)
    # by ~1e-2 within a few iterations: compare with the fp32-storage oracle, and bound the distance
    # from the fp64 oracle by twice that inherent spread (+1e-4)
    ref32 = osolver.ga_ngmres(_Fp32StorageFP(_SpectralA(grid, alpha, p), b, omega), np.zeros_like(b), w,
                              n_iter=iters, eps_rel=0.0, keep_iterates=True)
    ref32_res = [float(np.linalg.norm(fp.A @ x - b)) for x in ref32.iterates]
    spread = rel_l2(ref32.v, ref.v)
    err = rel_l2(host(v), ref.v)
    err32 = rel_l2(host(v), ref32.v)
    print(n, alpha, p, w, f"gpu vs oracle {err:.2e}, vs fp32-storage oracle {err32:.2e}, spread {spread:.2e}")
    print("res gpu", [f"{x:.3e}" for x in res])
    print("res ref", [f"{x:.3e}" for x in ref_res])
    assert err32 < 1e-3
    assert err < 1e-4 + 2 * spread
    # residual histories: the fp64 oracle's to 1e-4 until fp32 storage sets in (k < 4), then within
    # 1e-4 + twice the fp32-storage oracle's own deviation from it (two fp32 realisations of the same
    # iteration differ by rounding order, not only by storage)
    np.testing.assert_allclose(res[:4], ref_res[:4], rtol=1e-4)
    dev32 = max(abs(a - b) / b for a, b in zip(ref32_res, ref_res))
    np.testing.assert_allclose(res, ref_res, rtol=1e-4 + 2 * dev32, atol=1e-6 * ref_res[0])
    if w >= iters:  # NGMRES(infinity) = GMRES: residuals never increase
        assert all(res[k + 1] <= res[k] * (1 + 1e-5) for k in range(iters))
        assert res[-1] < 0.2 * res[0]
