"""Flow-map diagnostics (NEXT-2; figure captions; reading R32) on the GPU
vs the fp64 oracle: the displacement y - x to relative L2 1e-5; det(grad y) to 1e-5 of the
size of what it is made of — rms(det - 1) + rms(grad(y - x)) — plus the fp32 output
rounding at 1 (for a divergence-free v, det - 1 is a ~1e-6 cancellation of O(0.1)
derivatives); v = 0 gives the identity bitwise; a divergence-free v gives det ~ 1."""
import numpy as np
import pytest

from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import flowmap, spectral

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("cfg,n", [(1, (64, 64)), (2, (32, 32, 32)), (3, (32, 16, 64)), (4, (64, 64, 64))])
@pytest.mark.parametrize("scale", [0.5, 1.0])
def test_flow_map_matches_oracle(cfg, n, scale):
    d = case(cfg, n, scale=scale)
    t = topt_for(d)
    y, det = t.flow_map(dev(d["v"]))
    ry = flowmap.flow_map(d["grid"], d["v"], d["nt"])
    rdet = flowmap.det_grad(d["grid"], ry)
    assert rel_l2(host(y), ry) < TOL
    rms = lambda a: float(np.sqrt(np.mean(np.square(a))))
    rJ = np.stack([spectral.deriv(d["grid"], ry[b], a) for b in range(len(n)) for a in range(len(n))])
    assert rms(host(det) - rdet) <= TOL * (rms(rdet - 1.0) + rms(rJ)) + 2.0 ** -24
    assert host(det).min() > 0.0  # a diffeomorphism, as in the paper's figures


def test_flow_map_identity_and_incompressible():
    d = case(3, (32, 32, 32))
    t = topt_for(d)
    y, det = t.flow_map(dev(np.zeros_like(d["v"])))
    assert np.all(host(y) == 0.0) and np.all(host(det) == 1.0)
    vdf = spectral.leray(d["grid"], d["vstar"]).astype(np.float32).astype(np.float64)
    y, det = t.flow_map(dev(vdf))
    rdet = flowmap.det_grad(d["grid"], flowmap.flow_map(d["grid"], vdf, d["nt"]))
    assert np.max(np.abs(host(det) - 1.0)) < 2 * np.max(np.abs(rdet - 1.0)) + 1e-5
