"""Dev: run the FP32 (3xTF32 tcgen05) path on syn200 for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload
w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "syn200")
h = JKCals(w.T, w.R, hist_cap=20, precision=1)
h.set_init(w.P)
h.iterate(int(sys.argv[2]) if len(sys.argv) > 2 else 5, 0.0)
torch.cuda.synchronize()
print("done")
