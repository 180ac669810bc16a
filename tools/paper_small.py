"""The only absolute timings the paper prints: JK-CALS on the "small" tensor
50 x 100 x 100, R = 3 and R = 5, 100 iterations: 0.28 s / 0.27 s on 12 Xeon 8160 threads. Same
workload shape here (synthetic, seeded), FP64, one B200, device-timed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_pool, make_workload
out = []
for R in (3, 5, 7, 9):
    w = make_workload(((50, 100, 100), R, 5, 0.01, "syn", 100))
    h = JKCals(w.T, w.R, hist_cap=100)
    h.set_init(w.P); h.iterate(100, 0.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(h.stream); h.set_init(w.P); h.iterate(100, 0.0); e.record(h.stream); e.synchronize()
    print(f"small 50x100x100 R={R}: {s.elapsed_time(e):.2f} ms (100 iterations, 50 LOO submodels)")
w = make_pool("all_small")
h = JKCals(w.T, list(w.ranks), hist_cap=100)
h.set_init(w.Ps); h.iterate(100, 0.0)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(h.stream); h.set_init(w.Ps); h.iterate(100, 0.0); e.record(h.stream); e.synchronize()
print(f"small 'All' R in {{3,5,7,9}}: {s.elapsed_time(e):.2f} ms")
