import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from synth import make_workload
from paper_2112_03985_b200 import JKCals
for name, sweeps in [("4way", 1), ("4way", 5), ("4way", 20), ("syn200", 5)]:
    w = make_workload(name)
    ps = [0, 50]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=sweeps, nthreads=16)
    for prec in (0, 1):
        h = JKCals(w.T, w.R, hist_cap=sweeps, precision=prec)
        h.set_init(w.P); h.iterate(sweeps, 0.0)
        errs = []
        for q, p in enumerate(ps):
            fac, lam = h.factors(p)
            errs.append([float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(fac, res.factors[q])])
        print(name, sweeps, "fp32" if prec else "fp64", np.array(errs).max(axis=0))
