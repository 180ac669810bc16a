"""Dev: a few sweeps of one submodel shard (for ncu launch lists): shard_one.py <workload> <nsub> [sweeps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload

w = make_workload(sys.argv[1])
nsub = int(sys.argv[2])
sw = int(sys.argv[3]) if len(sys.argv) > 3 else 3
h = JKCals(w.T, w.R, hist_cap=sw, sub_range=(0, nsub))
h.set_init(w.P)
h.iterate(sw, 0.0)
torch.cuda.synchronize()
print("done")
