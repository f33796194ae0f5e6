"""Host-buffer entry points (end-to-end path of bench.py) against the device-buffer path:
the same kernels on the same inputs, so results must agree bitwise; consecutive streaming
calls alternate staging slots and must each return their own evaluation."""
import numpy as np
import pytest
import torch

from gpu_common import case, dev, topt_for

pytestmark = pytest.mark.gpu


def _pinned(x):
    return torch.tensor(np.asarray(x), dtype=torch.float32).pin_memory()


@pytest.mark.parametrize("cfg,n,model", [(2, (32, 32, 32), 1), (1, (64, 64), 0)])
def test_host_sync_and_streaming_match_device(cfg, n, model):
    d = case(cfg, n, model=model)
    t = topt_for(d)
    vs = [s * d["v"] for s in (0.5, 1.0, -0.7)]
    ref = []
    for v in vs:
        g, _, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(v))
        torch.cuda.synchronize()
        ref.append((g.cpu().numpy().copy(), sc.cpu().numpy().copy()))
    m0h, m1h = _pinned(d["m0"]), _pinned(d["m1"])
    # synchronous host call
    gh = torch.empty(vs[0].shape, dtype=torch.float32).pin_memory()
    sh = torch.zeros(16, dtype=torch.float64).pin_memory()
    t.eval_gradient_host(m0h, m1h, _pinned(vs[1]), gh, sh)
    assert np.array_equal(gh.numpy(), ref[1][0])
    assert np.array_equal(sh.numpy()[:7], ref[1][1][:7])
    # three streaming calls in flight (slots 0, 1, 0), one sync at the end
    vh = [_pinned(v) for v in vs]
    outs = [(torch.empty(v.shape, dtype=torch.float32).pin_memory(), torch.zeros(16, dtype=torch.float64).pin_memory())
            for v in vs]
    for v, (g_h, s_h) in zip(vh, outs):
        t.eval_gradient_host_async(m0h, m1h, v, g_h, s_h)
    torch.cuda.current_stream().synchronize()
    for (g_h, s_h), (gr, sr) in zip(outs, ref):
        assert np.array_equal(g_h.numpy(), gr)
        assert np.array_equal(s_h.numpy()[:7], sr[:7])
