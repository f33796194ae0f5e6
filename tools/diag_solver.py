import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import solver as osolver
d = case(4, (32, 32, 32), alpha=1e-4)
fp = osolver.TransportFP(d['prob'])
ls = osolver.LineSearchState()
v0 = np.zeros((3, 32, 32, 32))
ref = osolver.ga_ngmres(fp, v0, 3, 1, 0, 20, 0.0, 'ga', ls, keep_iterates=True)
print('oracle rhos', ls.accepted)
print('oracle rel', ['%.2e' % x for x in ref.rel_grad])
for k in [1, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20]:
    t = topt_for(d, window=3, sigma=1, tau=0, max_iter=k, eps_rel=0.0)
    v, rep = t.solve(dev(d['m0']), dev(d['m1']))
    tr = topt_for(d, window=3, sigma=1, tau=0, max_iter=k, eps_rel=0.0)
    tr.set_step_replay(ls.accepted)
    vr, repr_ = tr.solve(dev(d['m0']), dev(d['m1']))
    print(k, 'free: rho %.4g relv %.2e obj %.6e vs %.6e | replay relv %.2e gi %.3e vs %.3e' % (
        rep['rho'], rel_l2(host(v), ref.iterates[k]), rep['obj'], 0, rel_l2(host(vr), ref.iterates[k]),
        repr_['grad_inf'] / repr_['grad_inf0'], ref.rel_grad[k - 1]), flush=True)
