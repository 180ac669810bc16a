"""Full-size parity evidence: EVERY submodel of a BASELINE config on the GPU vs the oracle
(which fits each submodel on the explicitly sliced tensor), fixed sweeps. Slow (the oracle takes
minutes on the host cores), so it is a tool, not part of `pytest -m gpu`. Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2112_03985_b200 import JKCals
from synth import make_workload

name = sys.argv[1]
precs = [{"fp32": 1, "fp64_i8": 2}.get(x, 0) for x in (sys.argv[2] if len(sys.argv) > 2 else "fp64").split(",")]
w = make_workload(name)
t1 = time.time()
res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=os.cpu_count() or 1)
t2 = time.time()
for prec in precs:
    t0 = time.time()
    h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=prec)
    h.set_init(w.P)
    h.iterate(w.sweeps, 0.0)
    h.status()  # (synchronises)
    tg = time.time() - t0
    worst = [0.0] * len(w.dims)
    worst_lam, worst_err = 0.0, 0.0
    for p in range(w.dims[0]):
        fac, lam = h.factors(p)
        for n, (a, b) in enumerate(zip(fac, res.factors[p])):
            worst[n] = max(worst[n], float(np.linalg.norm(a - b) / np.linalg.norm(b)))
        worst_lam = max(worst_lam, float(np.linalg.norm(lam - res.lam[p]) / np.linalg.norm(res.lam[p])))
        hg, ho = h.history(p), res.history(p)
        worst_err = max(worst_err, float(np.max(np.abs(hg - ho) / np.abs(ho))))
    bar = 1e-4 if prec == 1 else 1e-10
    print(json.dumps({"config": name, "precision": ["fp64", "fp32", "fp64_i8"][prec], "submodels": w.dims[0],
                      "sweeps": w.sweeps, "worst_rel_factor_error_per_mode": worst, "worst_rel_lambda_error": worst_lam,
                      "worst_rel_error_history": worst_err, "bar": bar, "pass": max(worst + [worst_lam]) <= bar,
                      "gpu_s": round(tg, 2), "oracle_s": round(t2 - t1, 1), "oracle_threads": os.cpu_count(),
                      "round": 2}), flush=True)
    h.close()
