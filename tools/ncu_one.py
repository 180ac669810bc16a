"""Dev: a few eager sweeps of one config (for `ncu -k regex:... --launch-skip K --launch-count 1`)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "syn200"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = make_workload(name)
h = JKCals(w.T, w.R, hist_cap=sweeps, precision=prec)
h.set_init(w.P)
h.set_instrument(True)  # eager launches, one kernel per mode and step
h.iterate(sweeps, 0.0)
torch.cuda.synchronize()
print("done", name, sweeps)
