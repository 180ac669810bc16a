"""Dev: phase clocks of the cluster-resident kernel (build with -DJK_RES_PROF, JKCALS_LIB=...)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals
from paper_2112_03985_b200 import jkcals as J
from synth import make_workload

os.environ["JKCALS_RESIDENT"] = "1"
w = make_workload(sys.argv[1])
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 100
h = JKCals(w.T, w.R, hist_cap=sw)
h.set_init(w.P)
h.iterate(sw, 0.0)
h.set_init(w.P)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(h.stream); h.iterate(sw, 0.0); e.record(h.stream); e.synchronize()
out = np.zeros(8, dtype=np.int64)
L = J.lib()
L.jkcals_dev_res_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
L.jkcals_dev_res_prof(h._h, out.ctypes.data)
names = ["mttkrp", "ksplit-reduce", "cluster-sync1", "gather", "hadamard+chol", "solve..broadcast+error", "(owner loop end)", "cluster-sync2"]
tot = out.sum()
print(f"{sys.argv[1]}: {s.elapsed_time(e) / sw * 1e3:.1f} us/sweep; block 0 clocks per sweep:")
for nm, v in zip(names, out):
    print(f"  {nm:26s} {v / sw:10.0f} clk ({100 * v / max(tot, 1):5.1f} %)")
