"""Dev: FP32-path error on the fluorescence-shaped eem configs for a few submodels (env knobs:
JKCALS_TF32_PAIR, JKCALS_TF32_CHUNK), vs the FP64 oracle and vs the FP64 GPU path."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from synth import make_workload
from paper_2112_03985_b200 import JKCals

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

for name in sys.argv[1:] or ["eem_r5"]:
    w = make_workload(name)
    ps = [0, 100, 200, 267]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=os.cpu_count())
    h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=1)
    h.set_init(w.P); h.iterate(w.sweeps, 0.0)
    errs = {p: max(rel(a, b) for a, b in zip(h.factors(p)[0], res.factors[q])) for q, p in enumerate(ps)}
    # error after 1, 5, 20 sweeps (growth)
    grow = {}
    for sw in (1, 5, 20):
        r2 = O.jk_als(w.T, w.P, p_list=[0], max_iters=sw, nthreads=os.cpu_count())
        h.set_init(w.P); h.iterate(sw, 0.0)
        grow[sw] = max(rel(a, b) for a, b in zip(h.factors(0)[0], r2.factors[0]))
    print(json.dumps({"config": name, "pair": os.environ.get("JKCALS_TF32_PAIR", "1"),
                      "chunk": os.environ.get("JKCALS_TF32_CHUNK", "48"), "err100": errs, "growth_p0": grow}), flush=True)
