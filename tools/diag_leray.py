import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_common import dev, host, rel_l2
from oracle import spectral
from oracle.spectral import Grid
import paper_2510_08782_b200 as topt
for n in [(16,32,64),(16,16,16),(32,16,16),(16,32,32),(32,32,64),(64,32,16),(8,8,8),(16,8,8)]:
    g = Grid(n)
    t = topt.Topt(topt.Config(n=n, nt=4, alpha=1e-2, model=2), device='cuda:0')
    rng = np.random.default_rng(0)
    u = np.stack([spectral.gaussian_blur(g, rng.normal(size=g.shape), 2.0) for _ in range(3)]).astype(np.float32).astype(np.float64)
    out = host(t.leray(dev(u)))
    ref = spectral.leray(g, u)
    errs = [rel_l2(out[c], ref[c]) for c in range(3)]
    s = host(t.apply_precond(dev(u)))
    refs = -spectral.apply_inv_alpha_L(g, ref, 1e-2, 2)
    d = [rel_l2(host(t.derivative(dev(u[0]), a)), spectral.deriv(g, u[0], a)) for a in range(3)]
    # where is the error largest
    e = np.abs(out - ref); idx = np.unravel_index(np.argmax(e), e.shape)
    print(n, 'leray', ['%.2e' % x for x in errs], 'prec %.2e' % rel_l2(s, refs), 'deriv', ['%.1e' % x for x in d], 'argmax', idx, flush=True)
