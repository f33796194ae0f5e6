import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr, spectral
for cfg, n, model in [(5, (16, 32, 64), 1), (5, (16, 32, 64), 0), (2, (32, 32, 32), 1)]:
    d = case(cfg, n, model=model)
    t = topt_for(d)
    g, s, sc = t.eval_gradient(dev(d['m0']), dev(d['m1']), dev(d['v']))
    ref = ogr.evaluate(d['prob'], d['v'])
    lam, b = t.adjoint()
    lam, b = host(lam), host(b)
    traj = host(t.forward(dev(d['m0']), dev(d['v'])))
    print(cfg, n, model, 'm', ['%.1e' % rel_l2(traj[j], ref['m'][j]) for j in range(d['nt'] + 1)])
    print('   lam', ['%.1e' % rel_l2(lam[j], ref['lam'][j]) for j in range(d['nt'] + 1)])
    print('   b', ['%.2e' % rel_l2(b[c], ref['b'][c]) for c in range(3)], 'g %.2e s %.2e' % (rel_l2(host(g), ref['g']), rel_l2(host(s), ref['s'])))
    # derivative of the GPU lam vs oracle derivative of the same (GPU) lam
    for a in range(3):
        dl = host(t.derivative(dev(lam[4]), a))
        print('   dlam axis', a, '%.2e' % rel_l2(dl, spectral.deriv(d['grid'], lam[4].astype(np.float32).astype(np.float64), a)),
              ' grad err from lam err %.2e' % rel_l2(spectral.deriv(d['grid'], lam[4], a), spectral.deriv(d['grid'], ref['lam'][4], a)))
