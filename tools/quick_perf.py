"""Dev timing: JK-CALS sweep time and MTTKRP TFLOP/s per mode on one config (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals
from synth import POOLS, make_pool, make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "syn200"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prec = 1 if (len(sys.argv) > 3 and sys.argv[3] == "fp32") else 0
if name in POOLS:
    w = make_pool(name)
    w.R, w.P = list(w.ranks), w.Ps
    C = sum(w.ranks) * w.dims[0]
else:
    w = make_workload(name)
    C = w.R * w.dims[0]
h = JKCals(w.T, w.R, hist_cap=sweeps, precision=prec)
h.set_init(w.P); h.iterate(3, 0.0)
h.set_init(w.P)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(h.stream); h.iterate(sweeps, 0.0); e.record(h.stream); e.synchronize()
ms = s.elapsed_time(e)
fl = h.sweep_flops()
print(f"{name}{' fp32' if prec else ''}: {sweeps} sweeps {ms:.2f} ms, {ms/sweeps*1e3:.1f} us/sweep, MTTKRP-flop rate {fl*sweeps/(ms*1e-3)/1e12:.2f} TF/s")
h.set_init(w.P); h.set_instrument(True); h.iterate(10, 0.0)
tm, te, n = h.kernel_times()
P = float(np.prod(w.dims))
for m in range(len(w.dims)):
    f = 2 * C * P
    print(f"  mode {m}: mttkrp {tm[m]/10*1e3:.1f} us ({f/(tm[m]/10*1e-3)/1e12:.2f} TF/s), epilogue {te[m]/10*1e3:.1f} us")
