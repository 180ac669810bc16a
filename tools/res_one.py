"""Dev: one cluster-resident iterate of a small config (for ncu -k regex:resident)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload

os.environ["JKCALS_RESIDENT"] = "1"
w = make_workload(sys.argv[1])
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = JKCals(w.T, w.R, hist_cap=sw)
h.set_init(w.P)
h.iterate(sw, 0.0)
torch.cuda.synchronize()
print("done")
