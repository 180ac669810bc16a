"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family on tiny shapes (FP64 LOO + tol compaction, delete-d pool, alignment, migration,
FP32 path, stand-alone MTTKRP)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals, mttkrp
from synth import make_pool, make_workload

w = make_workload("tiny")
h = JKCals(w.T, w.R, hist_cap=20, spare=2)
h.set_init(w.P)
h.iterate(5, 0.0)
h.iterate(40, 1e-6)
h.align()
h.aligned_stats(1)
h.jackknife_stats(1)
for m in range(3):
    h.all_factors(m)
p = make_pool(((12, 7, 5), (2, 3), 3, 0.01, "syn", 10), seed=1)
hp = JKCals(p.T, list(p.ranks), hist_cap=10, d=5, spare=1)
hp.set_init(p.Ps)
hp.iterate(6, 0.0)
hb = JKCals(p.T, list(p.ranks), sub_range=(0, 1), hist_cap=10, d=5, spare=2)
hb.set_init(p.Ps)
hb.iterate(6, 0.0)
hb.import_submodel(hp.export_submodel(4))
hp.iterate(4, 0.0)
hb.iterate(4, 0.0)
hp.align()
h32 = JKCals(w.T, w.R, hist_cap=10, precision=1)
h32.set_init(w.P)
h32.iterate(5, 0.0)
# r02 kernels: FP32 CTA pairs with an odd tile count + 4 j' per k-tile, the cluster-resident
# syn50-size path, tol mode through the CUDA-graph WHILE node
w6 = make_workload(((60, 44, 36), 6, 6, 0.01, "syn", 4))
h6 = JKCals(w6.T, w6.R, hist_cap=4, precision=1)
h6.set_init(w6.P)
h6.iterate(3, 0.0)
w1 = make_workload("syn50_r1")
hr = JKCals(w1.T, w1.R, hist_cap=8)
hr.set_init(w1.P)
hr.iterate(4, 0.0)
w3 = make_workload("syn50_r3")
os.environ["JKCALS_RESIDENT"] = "0"
ht = JKCals(w3.T, w3.R, hist_cap=200)
ht.set_init(w3.P)
ht.iterate(200, 1e-6)
g = np.random.default_rng(0)
dims, C = (9, 7, 5), 20
T = torch.from_numpy(g.standard_normal(int(np.prod(dims)))).cuda()
U = [torch.from_numpy(np.pad(g.standard_normal((I, C)), ((0, 0), (0, 108)))).cuda() for I in dims]
for n in range(3):
    mttkrp(T, dims, n, U, C)
torch.cuda.synchronize()
print("sanitize workload done")
