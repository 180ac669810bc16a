"""Dev: time one INT8-sliced MTTKRP (syn200 shape, mode 1) -- run under JKCALS_I8_PROBE=0/1/2 to
split the kernel time into MMA+TMA (probe 1 skips the drain) and drain+TMA (probe 2 issues one
product per K32 step). Probe results are wrong by construction; only the time is read."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200.jkcals import mttkrp_i8
g = np.random.default_rng(1)
dims, C = (200, 200, 200), 1000
Td = torch.from_numpy(g.uniform(0, 1, int(np.prod(dims)))).cuda()
Ud = [torch.from_numpy(np.pad(g.uniform(0, 1, (I, C)), ((0, 0), (0, 24)))).cuda() for I in dims]
for _ in range(3):
    mttkrp_i8(Td, dims, 1, Ud, C)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    mttkrp_i8(Td, dims, 1, Ud, C)
e.record()
e.synchronize()
print("probe", os.environ.get("JKCALS_I8_PROBE", "0"), "ms per call (incl. slicing + reduce)", s.elapsed_time(e) / 20)
