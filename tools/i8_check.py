"""Dev: the experimental INT8-sliced MTTKRP vs the oracle (relative error) and its kernel time vs
the DMMA MTTKRP, on a few shapes incl. syn200 (FP64-equivalent TFLOP/s of 2 C prod(I))."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2112_03985_b200 import mttkrp
from paper_2112_03985_b200.jkcals import mttkrp_i8

g = np.random.default_rng(1)
for dims, C, check in (((10, 8, 6), 20, True), ((37, 23, 11), 129, True), ((13, 7, 5, 3), 70, True),
                       ((50, 50, 50), 250, True), ((200, 200, 200), 1000, False)):
    T = np.asfortranarray(g.uniform(0, 1, dims))
    U = [g.uniform(0, 1, (I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(len(dims)):
        Mi = mttkrp_i8(Td, dims, n, Ud, C)
        Md = mttkrp(Td, dims, n, Ud, C)
        torch.cuda.synchronize()
        line = f"{dims} C={C} n={n}: i8 vs dmma rel {float(torch.linalg.norm(Mi - Md) / torch.linalg.norm(Md)):.2e}"
        if check:
            ref = O.mttkrp(T, U, n)
            line += f", i8 vs oracle {np.linalg.norm(Mi.cpu().numpy() - ref) / np.linalg.norm(ref):.2e}"
            line += f", dmma vs oracle {np.linalg.norm(Md.cpu().numpy() - ref) / np.linalg.norm(ref):.2e}"
        print(line, flush=True)
        if not check and n == 0:
            for f, nm in ((mttkrp_i8, "i8 (incl. operand slicing)"), (mttkrp, "dmma")):
                f(Td, dims, n, Ud, C)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(3):
                    f(Td, dims, n, Ud, C)
                e.record()
                e.synchronize()
                ms = s.elapsed_time(e) / 3
                print(f"  {nm}: {ms:.3f} ms per call = {2 * C * np.prod(dims) / (ms * 1e-3) / 1e12:.1f} TF/s", flush=True)
