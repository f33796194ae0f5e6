"""Race stress and device bounds checks (substitute for compute-sanitizer racecheck / synccheck /
memcheck, which is closed on this GPU pool: "runs under it have left GPUs needing a reset").

libtopt_stress.so is the same sources built with -DTOPT_STRESS (csrc/internal.cuh): at every
synchronisation point of the pipelined kernels — the SL plane ring's refill barrier, the trace's
pair barrier, the TMA slot waits and releases of the body force, the staging barrier of the merged
last-axis pass, and both sides of every line-FFT exchange — a pseudo-random quarter of the warps
sleeps up to ~1 us (seeded by the clock), and ring / window indices are checked with __trap().  A
missing barrier, an early refill or a wrong mbarrier phase then changes results or traps.  Every
kernel's arithmetic is order-fixed, so each evaluation must be BITWISE identical to the release
library's, run after run.  The stress library runs in a subprocess (its own CUDA context)."""
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
digest = lambda *ts: hashlib.sha256(b"".join(t.cpu().numpy().tobytes() for t in ts)).hexdigest()
out = {}
for cfg, n, model, world, scale in json.loads(sys.argv[2]):
    d = case(cfg, tuple(n), model=model, scale=scale)
    t = topt_for(d, world=world, max_iter=3, eps_rel=0.0)
    hs = []
    for rep in range(2):  # two evaluations: identical to each other
        g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
        torch.cuda.synchronize()
        hs.append(digest(g, s, sc))
    v, r = t.solve(dev(d["m0"]), dev(d["m1"]))
    torch.cuda.synchronize()
    out[f"{cfg}-{n}-{model}-{world}-{scale}"] = [hs[0], hs[1], digest(v), r["obj"]]
print("RESULT " + json.dumps(out))
"""


def _run(lib, cases):
    env = dict(os.environ)
    if lib:
        env["TOPT_LIB"] = lib
    p = subprocess.run([sys.executable, "-c", _WORKER, ROOT, json.dumps(cases)], capture_output=True, text=True,
                       env=env, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")][-1]
    return json.loads(line[7:])


def test_stress_library_is_bitwise_identical():
    assert os.path.exists(STRESS), "build() writes libtopt_stress.so"
    cases = [[c, list(n), m, w, 1.0] for c, n, m, w in CASES]
    cases.append([2, [64, 32, 32], 1, 2, 4.0])  # feet beyond the halo: the z-slab window path
    ref = _run(None, cases)
    for rep in range(2):
        got = _run(STRESS, cases)
        for k in ref:
            assert got[k][0] == got[k][1], (k, "stress: two evaluations differ")
            assert got[k][:3] == ref[k][:3], (k, rep, "stress build differs from release")
            assert got[k][3] == ref[k][3], k
