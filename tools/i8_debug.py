"""Dev: where does the INT8-sliced MTTKRP differ from the oracle (per tile row i mod kI8N)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_03985_b200.jkcals import mttkrp_i8
from oracle import oracle as O
for dims, C in [((10, 8, 6), 20), ((200, 50, 20), 130)]:
    g = np.random.default_rng(3)
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(3):
        M = mttkrp_i8(Td, dims, n, Ud, C).cpu().numpy()
        ref = O.mttkrp(T, U, n)
        err = np.abs(M - ref) / np.abs(ref).max()
        rows = err.max(axis=1)
        print(dims, C, n, "max", err.max(), "bad rows (i mod 80):", sorted(set((np.nonzero(rows > 1e-12)[0] % 80).tolist()))[:40],
              "bad cols:", len(np.nonzero(err.max(axis=0) > 1e-12)[0]), "ratio", np.median(M[rows > 1e-12] / ref[rows > 1e-12]) if (rows > 1e-12).any() else None)
