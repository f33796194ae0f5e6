"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel of
libtopt at 64^3 (and the SL plane ring and the trace at 128^3), through the public C ABI.

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py [--big]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gpu_common import case, dev, topt_for  # noqa: E402
from oracle import spectral  # noqa: E402


def main():
    big = "--big" in sys.argv
    if big:  # the SL plane ring (STEP / LAST / EFACTOR) and the trace at 128^3
        d = case(3, (128, 128, 128), model=1)
        t = topt_for(d)
        t.feet(dev(d["v"]))
        t.forward(dev(d["m0"]), dev(d["v"]))
        t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
        torch.cuda.synchronize()
        print("sanitize --big: done")
        return
    for cfg, n in ((2, (64, 64, 64)), (1, (64, 64)), (2, (8, 8, 8))):
        for model in (0, 1, 2):
            d = case(cfg, n, model=model)
            if model == 2:
                d["v"] = spectral.leray(d["grid"], d["v"]).astype(np.float32).astype(np.float64)
            t = topt_for(d, max_iter=3, eps_rel=0.0)
            m0, m1, v = dev(d["m0"]), dev(d["m1"]), dev(d["v"])
            t.eval_gradient(m0, m1, v)
            t.adjoint()
            t.feet(v)
            t.forward(m0, v)
            t.objective(m0, m1, v)
            for a in range(len(n)):
                t.derivative(m0, a)
            t.apply_precond(v)
            t.leray(v)
            t.multidot(v, [v, v, v])
            t.mix(v, [v, v], [0.5, -0.25])
            t.solve(m0, m1)
            if model == 0:
                t.flow_map(v)
                hm0, hm1, hv = (x.cpu().pin_memory() for x in (m0, m1, v))
                hg = torch.empty_like(hv).pin_memory()
                hs = torch.zeros(16, dtype=torch.float64).pin_memory()
                for _ in range(3):
                    t.eval_gradient_host_async(hm0, hm1, hv, hg, hs)
                t.eval_gradient_host(hm0, hm1, hv, hg, hs)
            torch.cuda.synchronize()
    # large displacements: per-point stencils and the L1 fallback inside the tiled kernels
    d = case(2, (64, 32, 32), scale=4.0)
    t = topt_for(d)
    t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
    # emulated z-slabs, both transports
    for transport in ("nccl", "p2p"):
        for model in (0, 1, 2):
            d = case(2, (64, 32, 32), model=model)
            tp = topt_for(d, world=2, max_iter=2, eps_rel=0.0)
            tp.set_transport(transport)
            tp.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
            tp.solve(dev(d["m0"]), dev(d["m1"]))
    torch.cuda.synchronize()
    print("sanitize: done")


if __name__ == "__main__":
    main()
