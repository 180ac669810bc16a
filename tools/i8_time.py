"""Dev: kernels of one experimental INT8-sliced MTTKRP call on syn200's shape (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import mttkrp
from paper_2112_03985_b200.jkcals import mttkrp_i8
g = np.random.default_rng(1)
dims, C = (200, 200, 200), 1000
Td = torch.from_numpy(g.uniform(0, 1, int(np.prod(dims)))).cuda()
Ud = [torch.from_numpy(np.pad(g.uniform(0, 1, (I, C)), ((0, 0), (0, 24)))).cuda() for I in dims]
for n in (1, 0):
    mttkrp_i8(Td, dims, n, Ud, C)
    mttkrp(Td, dims, n, Ud, C)
torch.cuda.synchronize()
print("done")
