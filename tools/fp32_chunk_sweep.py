"""Dev: FP32-path chunk length vs accuracy (4 submodels vs the oracle after 100 sweeps) and time
(100 sweeps) on one config; JKCALS_TF32_CHUNK is read once per process, so each value runs in a child."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
from oracle import oracle as O
from synth import make_workload
from paper_2112_03985_b200 import JKCals
w = make_workload(sys.argv[1])
ps = [0, w.dims[0] // 3, 2 * w.dims[0] // 3, w.dims[0] - 1]
h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=1)
h.set_init(w.P); h.iterate(3, 0.0); h.set_init(w.P)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(h.stream); h.iterate(w.sweeps, 0.0); e.record(h.stream); e.synchronize()
res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=os.cpu_count())
err = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for q, p in enumerate(ps) for a, b in zip(h.factors(p)[0], res.factors[q]))
print(json.dumps({"ms": round(s.elapsed_time(e), 2), "err": err}))
""" % ROOT
cfg = sys.argv[1]
for ch in sys.argv[2:]:
    env = dict(os.environ, JKCALS_TF32_CHUNK=ch)
    out = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.returncode == 0 else json.dumps({"err": out.stderr[-300:]})
    print(json.dumps({"config": cfg, "chunk": int(ch), **json.loads(line)}), flush=True)
