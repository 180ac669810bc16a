"""The paper's second application shape: a 44 x 2700 x 200 tensor, three
models of ranks {19, 20, 21} jackknifed together (the "All" group), FP64. Synthetic data of that
shape (the real dataset is out of scope). Reports the fixed-sweep time and a tol = 1e-6 run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals
from synth import make_pool

w = make_pool(((44, 2700, 200), (19, 20, 21), 20, 0.01, "syn", 100), seed=0)
h = JKCals(w.T, list(w.ranks), hist_cap=1000)
h.set_init(w.Ps); h.iterate(3, 0.0)
for sweeps, tol in ((100, 0.0), (1000, 1e-6)):
    h.set_init(w.Ps)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(h.stream); done = h.iterate(sweeps, tol); e.record(h.stream); e.synchronize()
    st = h.status()
    print(f"44x2700x200 pool R in {{19,20,21}} (132 submodels, C = 2640): tol={tol:g} "
          f"{s.elapsed_time(e):.1f} ms for {done} sweeps; iterations min/median/max "
          f"{st['iters'].min()}/{int(np.median(st['iters']))}/{st['iters'].max()}")
h.set_init(w.Ps); h.set_instrument(True); h.iterate(5, 0.0)
tm, te, n = h.kernel_times()
print("per mode: mttkrp us", [round(x / 5 * 1e3, 1) for x in tm], "epilogue us", [round(x / 5 * 1e3, 1) for x in te])
