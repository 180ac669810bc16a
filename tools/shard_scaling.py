"""Dev: predicted strong scaling of the syn200 bench -- time one rank's shard (sub_range of
200/G submodels) on one GPU for G = 1, 2, 4, 8 (ranks are independent: no per-sweep comms)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from paper_2112_03985_b200.dist import shard
from synth import make_workload

w = make_workload("syn200")
Td = torch.from_numpy(w.T.ravel(order="F").copy()).cuda()
t1 = None
for G in (1, 2, 4, 8):
    worst = 0.0
    for r in sorted({0, G - 1}):
        a, b = shard(200, G, r)
        h = JKCals(Td, w.R, sub_range=(a, b), hist_cap=100, dims=w.dims)
        h.set_init(w.P); h.iterate(100, 0.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(h.stream); h.set_init(w.P); h.iterate(100, 0.0); e.record(h.stream); e.synchronize()
        worst = max(worst, s.elapsed_time(e))
        h.close()
    t1 = t1 or worst
    print(f"G={G}: per-rank {worst:.2f} ms, predicted efficiency {t1 / (G * worst):.3f}")

# per-mode breakdown of the G = 8 shard (instrumented eager launches)
for G in (4, 8):
    a, b = shard(200, G, 0)
    h = JKCals(Td, w.R, sub_range=(a, b), hist_cap=100, dims=w.dims)
    h.set_init(w.P); h.set_instrument(True); h.iterate(20, 0.0)
    tm, te, n = h.kernel_times()
    print(f"G={G} shard [{a},{b}): mttkrp us/mode", [round(x / 20 * 1e3, 1) for x in tm],
          "epilogue us/mode", [round(x / 20 * 1e3, 1) for x in te])
