"""Dev: FP32 path bitwise determinism (two runs of the same job)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2112_03985_b200 import JKCals
from synth import make_workload
for name in ("syn50_r5", "eem_r5"):
    w = make_workload(name)
    out = []
    for rep in range(2):
        h = JKCals(w.T, w.R, hist_cap=10, precision=1)
        h.set_init(w.P); h.iterate(10, 0.0)
        out.append(np.concatenate([np.ravel(f) for p in (0, 7, w.dims[0] - 1) for f in h.factors(p)[0]]))
        h.close()
    print(name, "bitwise equal:", bool(np.array_equal(out[0], out[1])))
