"""Tolerance-mode wall time: WHILE-graph device trigger vs the per-sweep host check.

Run twice, with and without JKCALS_TOL_HOST_LOOP=1 (read once per process). Prints one JSON line per
workload: seconds for iterate(1000, tol=1e-6) (median of 3 after a warm-up, factors re-initialised
each time) and the sweeps run.
"""
import json, os, sys, time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_03985_b200 import JKCals  # noqa: E402
from synth import make_workload  # noqa: E402

os.environ.setdefault("JKCALS_RESIDENT", "0")  # the streamed path (where the trigger applies)
for name in sys.argv[1:] or ["syn50_r3", "syn50_r5", "eem_r5"]:
    w = make_workload(name)
    h = JKCals(w.T, w.R, hist_cap=1000)
    ts, done = [], 0
    for rep in range(4):
        h.set_init(w.P)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        done = h.iterate(1000, 1e-6)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"workload": name, "host_loop": os.environ.get("JKCALS_TOL_HOST_LOOP", "0"),
                      "s": round(float(np.median(ts[1:])), 5), "sweeps": done}), flush=True)
