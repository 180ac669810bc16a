"""Dev: FP32-path time and accuracy at the current JKCALS_TF32_CHUNK (read once per process):
syn200, 100 timed sweeps; factor error vs the FP64 oracle after 5 sweeps for submodels {0, 100}."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2112_03985_b200 import JKCals
from synth import make_workload

w = make_workload("syn200")
h = JKCals(w.T, w.R, hist_cap=100, precision=1)
h.set_init(w.P); h.iterate(3, 0.0); h.set_init(w.P)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(h.stream); h.iterate(100, 0.0); e.record(h.stream); e.synchronize()
ms = s.elapsed_time(e)
ps = [0, 100]
res = O.jk_als(w.T, w.P, p_list=ps, max_iters=5, nthreads=os.cpu_count())
h.set_init(w.P); h.iterate(5, 0.0)
err = max(float(np.linalg.norm(a - b) / np.linalg.norm(b))
          for q, p in enumerate(ps) for a, b in zip(h.factors(p)[0], res.factors[q]))
print(json.dumps({"chunk": os.environ.get("JKCALS_TF32_CHUNK", "48"), "ms_100": round(ms, 2), "err5": err}), flush=True)
