"""Dev: MTTKRP time of the FP64_I8 sweep path on syn200 -- run under JKCALS_I8_PROBE=0/1/2 to split
the INT8 kernel time into MMA+TMA (probe 1 skips the drain) and drain+TMA (probe 2 issues one
product per K32 step). Probe results are wrong by construction; only the time is read."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload
w = make_workload("syn200")
h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=2)
h.set_init(w.P)
h.iterate(5, 0.0)
h.set_instrument(True)
h.iterate(10, 0.0)
tm, te, nl = h.kernel_times()
print("probe", os.environ.get("JKCALS_I8_PROBE", "0"), "MTTKRP ms per mode (slice U + i8 kernel)", float(tm.sum()) / nl,
      "epilogue", float(te.sum()) / nl)
