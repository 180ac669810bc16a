"""Dev probe: the epilogue's %globaltimer phase stamps (-DJK_EPI_PROF, printed by blocks 0 and K-1).

Build once here (the dev library lands in paper_2112_03985_b200/build/, which travels to the GPU box):
    JKCALS_BUILD_LIB=$PWD/paper_2112_03985_b200/build/libjkcals_epiprof.so JKCALS_NVCC_EXTRA=-DJK_EPI_PROF \\
        python -c "from paper_2112_03985_b200 import _build; _build.build()"
then on the GPU: python tools/epi_prof.py <workload> [nsub]
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["JKCALS_LIB"] = os.path.join(ROOT, "paper_2112_03985_b200", "build", "libjkcals_epiprof.so")
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload
w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "syn200")
nsub = int(sys.argv[2]) if len(sys.argv) > 2 else w.dims[0]
os.environ.setdefault("JKCALS_RESIDENT", "0")
h = JKCals(w.T, w.R, hist_cap=10, sub_range=(0, nsub))
h.set_init(w.P)
h.set_instrument(True)  # eager launches: the printf output of each epilogue in order
h.iterate(2, 0.0)
torch.cuda.synchronize()
