"""g and s of the merged v/b chain vs the oracle across grid sizes (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from gpu_common import case, dev, host, rel_l2, topt_for
from oracle import gradient as ogr

for cfg, n in [(2, (8, 8, 8)), (2, (16, 16, 16)), (2, (32, 32, 32)), (2, (64, 16, 8)), (3, (32, 16, 64)), (1, (64, 64)), (1, (8, 8))]:
    for model in (0, 1):
        d = case(cfg, n, model=model, scale=0.25)
        t = topt_for(d)
        g, s, sc = t.eval_gradient(dev(d["m0"]), dev(d["m1"]), dev(d["v"]))
        ref = ogr.evaluate(d["prob"], d["v"])
        sd = t.scalars_dict(sc)
        print(n, model, "g", rel_l2(host(g), ref["g"]), "s", rel_l2(host(s), ref["s"]), "reg", sd["reg"] / ref["reg"] - 1,
              "gs", sd["gs"] / ref["gs"] - 1, "slv", sd["slv"], flush=True)
