"""Race stress and device bounds checks (substitute for compute-sanitizer racecheck / synccheck /
memcheck, which is closed on this GPU pool: "runs under it have left GPUs needing a reset").

libtopt_stress.so is the same sources built with -DTOPT_STRESS (csrc/internal.cuh): at every
synchronisation point of the pipelined kernels — the SL plane ring's refill barrier, the trace's
pair barrier, the TMA slot waits and releases of the body force, the staging barrier of the merged
last-axis pass, and both sides of every line-FFT exchange — a pseudo-random quarter of the warps
sleeps up to ~1 us (seeded by the clock), and ring / window indices are checked with __trap().  A
missing barrier, an early refill or a wrong mbarrier phase then changes results or traps.  Every
kernel's arithmetic is order-fixed, so the stressed library must reproduce ITSELF bitwise from one
process to the next (each process draws other delays) and within a process; against the release
library it agrees to 1e-6 (not bitwise: the inserted delay points change the compiler's FMA
contraction in the assembly — measured 1.3e-7 relative in s, g bitwise equal).  The stress library
runs in subprocesses (their own CUDA contexts)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRESS = os.path.join(ROOT, "paper_2510_08782_b200", "lib", "libtopt_stress.so")

# (config recipe, grid, model, world): tiled SL kernels, line FFTs of every length used, the merged
# chain (one slab), Leray chains (incompressible), and emulated z-slabs (halo, window, transposes)
CASES = [(2, (64, 64, 64), 0, 1), (4, (64, 64, 64), 1, 1), (3, (32, 16, 64), 2, 1), (2, (64, 32, 32), 1, 2),
         (1, (64, 64), 0, 1), (2, (64, 32, 32), 0, 4)]

_WORKER = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from gpu_common import case, dev, topt_for
arrs, out = {}, {}
for i, (cfg, n, model, world, scale) in enumerate(json.loads(sys.argv[2])):
    d = case(cfg, tuple(n), model=model, scale=scale)
    t = topt_for(d, world=world, max_iter=3, eps_rel=0.0)
    hs = []
    for rep in range(2):  # two evaluations: identical to each other
        g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
        torch.cuda.synchronize()
        hs.append(hashlib.sha256(g.cpu().numpy().tobytes() + s.cpu().numpy().tobytes()).hexdigest())
    v, r = t.solve(dev(d["m0"]), dev(d["m1"]))
    torch.cuda.synchronize()
    arrs[f"g{i}"], arrs[f"s{i}"], arrs[f"v{i}"] = g.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
    out[str(i)] = hs + [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest(), r["obj"]]
np.savez(sys.argv[3], **arrs)
print("RESULT " + json.dumps(out))
"""


def _run(lib, cases, path):
    env = dict(os.environ)
    if lib:
        env["TOPT_LIB"] = lib
    p = subprocess.run([sys.executable, "-c", _WORKER, ROOT, json.dumps(cases), path], capture_output=True,
                       text=True, env=env, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")][-1]
    return json.loads(line[7:]), dict(np.load(path))


def test_stress_library_reproduces_itself_and_the_release(tmp_path):
    assert os.path.exists(STRESS), "build() writes libtopt_stress.so"
    cases = [[c, list(n), m, w, 1.0] for c, n, m, w in CASES]
    cases.append([2, [64, 32, 32], 1, 2, 4.0])  # feet beyond the halo: the z-slab window path
    ref, ra = _run(None, cases, str(tmp_path / "rel.npz"))
    s1, a1 = _run(STRESS, cases, str(tmp_path / "s1.npz"))
    s2, a2 = _run(STRESS, cases, str(tmp_path / "s2.npz"))
    for k in ref:
        assert s1[k][0] == s1[k][1] and s2[k][0] == s2[k][1], (k, "two evaluations in one process differ")
        assert s1[k] == s2[k], (k, "two stressed processes differ: a race")
    for name in ra:
        den = float(np.max(np.abs(ra[name]))) or 1.0
        assert float(np.max(np.abs(ra[name].astype(np.float64) - a1[name]))) <= 1e-6 * den, name
