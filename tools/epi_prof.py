"""Dev probe: build libjkcals with -DJK_EPI_PROF (globaltimer phase stamps in the epilogue,
printed by blocks 0 and K-1) into /tmp and run a few sweeps of one config."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_03985_b200 import _build
lib = "/tmp/libjkcals_dbg.so"
subprocess.check_call([_build.NVCC, *_build.FLAGS, "-DJK_EPI_PROF", "-o", lib,
                       os.path.join(_build.HERE, "csrc", "jkcals.cu")])
_build.LIB = lib
_build.stale = lambda: False
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload
w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "syn200")
nsub = int(sys.argv[2]) if len(sys.argv) > 2 else w.dims[0]
h = JKCals(w.T, w.R, hist_cap=10, sub_range=(0, nsub))
h.set_init(w.P)
h.iterate(2, 0.0)
torch.cuda.synchronize()
