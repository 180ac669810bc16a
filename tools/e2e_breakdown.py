"""Dev: where the end-to-end (host buffers) time of one syn200 job goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload

w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "syn200")
pin = torch.empty(w.T.size, dtype=torch.float64, pin_memory=True)
pin.numpy()[:] = np.ravel(w.T, order="F")
Pp = []
for p in w.P:
    t = torch.empty(p.size, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = np.ravel(p, order="F")
    Pp.append(t.numpy().reshape(p.shape, order="F"))
for rep in range(3):
    for label, T, P in (("pageable", w.T, w.P), ("pinned", pin.numpy(), Pp)):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        h = JKCals(T, w.R, hist_cap=w.sweeps, dims=w.dims); torch.cuda.synchronize(); t.append(time.perf_counter())
        h.set_init(P); torch.cuda.synchronize(); t.append(time.perf_counter())
        h.iterate(1, 0.0); torch.cuda.synchronize(); t.append(time.perf_counter())
        h.iterate(w.sweeps - 1, 0.0); torch.cuda.synchronize(); t.append(time.perf_counter())
        for m in range(3):
            h.all_factors(m)
        for m in range(1, 3):
            h.local_moments(m)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        h.close(); t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        print(f"{label:9s} create {d[0]:.2f} ms, set_init {d[1]:.2f}, sweep1(+capture) {d[2]:.2f}, "
              f"sweeps {d[3]:.2f}, outputs {d[4]:.2f}, close {d[5]:.2f}; total {sum(d):.2f}")
