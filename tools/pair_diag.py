"""Dev: FP32-path error vs the oracle for a few custom shapes (pair vs one-CTA via JKCALS_TF32_PAIR)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from synth import make_workload
from paper_2112_03985_b200 import JKCals

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

for spec in [((60, 44, 36), 6, 5, 0.01, "syn", 30), ((60, 44, 36), 6, 6, 0.01, "syn", 30),
             ((60, 48, 40), 5, 5, 0.01, "syn", 30), ((50, 50, 50), 5, 5, 0.01, "syn", 30)]:
    w = make_workload(spec)
    ps = [0, 31, 49]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=os.cpu_count())
    h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=1)
    h.set_init(w.P); h.iterate(w.sweeps, 0.0)
    worst = max(rel(a, b) for q, p in enumerate(ps) for a, b in zip(h.factors(p)[0], res.factors[q]))
    print(json.dumps({"spec": str(spec[:3]), "pair": os.environ.get("JKCALS_TF32_PAIR", "1"), "err": worst}), flush=True)
