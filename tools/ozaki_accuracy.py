"""CPU study for the next-round INT8-sliced FP64 MTTKRP: emulate the scheme
exactly in numpy (balanced base-128 digits, per-row / per-column power-of-two scales, only the
products whose digit indices sum to <= S-1, exact integer accumulation) and measure
(1) the MTTKRP error vs FP64, (2) the final JK-CALS factor error vs the oracle after full
sweeps when every MTTKRP of the ALS loop uses the emulation.  Usage: ozaki_accuracy.py [S]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from synth import make_workload

S = int(sys.argv[1]) if len(sys.argv) > 1 else 7


def digits(X, axis_scale):
    """X (2-D) -> (list of S int64 digit arrays, scale exponents along `axis_scale`):
    X = 2^e * sum_s d_s 2^(-7(s+1)) with |X 2^-e| <= 1/2, balanced digits |d| <= 64."""
    m = np.max(np.abs(X), axis=axis_scale, keepdims=True)
    e = np.where(m > 0, np.ceil(np.log2(np.where(m > 0, m, 1.0))) + 1, 0).astype(np.int64)
    r = X * np.exp2(-e.astype(np.float64))
    ds = []
    for _ in range(S):
        r = r * 128.0
        d = np.rint(r)
        ds.append(d.astype(np.int64))
        r = r - d
    return ds, e


def mttkrp_emulated(Tn, K):
    """Tn (I x J) @ K (J x C) with the INT8-sliced scheme."""
    A, ea = digits(Tn, 1)   # per-row scale of T_(n)
    B, eb = digits(K, 0)    # per-column scale of the KRP
    acc = np.zeros((Tn.shape[0], K.shape[1]))
    for d in range(S - 1, -1, -1):          # small terms first
        Dd = np.zeros((Tn.shape[0], K.shape[1]), dtype=np.int64)
        for a in range(d + 1):
            Dd += A[a] @ B[d - a]            # exact integer products
        acc += Dd.astype(np.float64) * 2.0 ** (-7 * (d + 2))
    return acc * np.exp2(ea.astype(np.float64)) * np.exp2(eb.astype(np.float64))


def unfold(T, n):
    return np.reshape(np.moveaxis(T, n, 0), (T.shape[n], -1), order="F")


def krp(mats):
    R = mats[0].shape[1]
    cols = []
    for r in range(R):
        c = np.ones(1)
        for m in mats:
            c = np.kron(m[:, r], c)
        cols.append(c)
    return np.stack(cols, axis=1)


def jk_cals(T, P, sweeps, emulate):
    dims = T.shape
    N, I0, R = len(dims), dims[0], P[0].shape[1]
    U = [p.copy() for p in P]
    Ub = [[u.copy() for u in U] for _ in range(I0)]
    for p in range(I0):
        Ub[p][0][p] = 0.0
    for it in range(sweeps):
        for n in range(N):
            # the fused multi-factor: all submodels' blocks side by side (one MTTKRP per mode)
            rest = [m for m in range(N) if m != n]
            K = np.concatenate([krp([Ub[p][m] for m in rest]) for p in range(I0)], axis=1)
            Mall = mttkrp_emulated(unfold(T, n), K) if emulate else unfold(T, n) @ K
            for p in range(I0):
                M = Mall[:, p * R:(p + 1) * R]
                H = np.ones((R, R))
                for m in rest:
                    H *= Ub[p][m].T @ Ub[p][m]
                V = np.linalg.solve(H, M.T).T
                if n == 0:
                    V[p] = 0.0
                Ub[p][n] = V / np.linalg.norm(V, axis=0)
    return Ub


for name, sweeps in (("tiny", 50), ("syn50_r3", 30), ("eem-like 40x30x20 R4", 30)):
    w = make_workload(((40, 30, 20), 4, 5, 0.02, "eem", 30), seed=1) if name.startswith("eem") else make_workload(name)
    T = np.asarray(w.T)
    rest = [1, 2]
    K = krp([w.P[m] for m in rest])
    M = unfold(T, 0) @ K
    Me = mttkrp_emulated(unfold(T, 0), K)
    print(f"{name}: S = {S} single MTTKRP relative error {np.linalg.norm(Me - M) / np.linalg.norm(M):.2e}")
    res = O.jk_als(w.T, w.P, max_iters=sweeps)
    Ue = jk_cals(T, w.P, sweeps, emulate=True)
    worst = 0.0
    for p in range(w.dims[0]):
        for n in range(3):
            a = np.delete(Ue[p][0], p, axis=0) if n == 0 else Ue[p][n]
            b = res.factors[p][n]
            worst = max(worst, np.linalg.norm(a - b) / np.linalg.norm(b))
    print(f"{name}: S = {S}, {sweeps} sweeps, worst relative factor error vs the oracle {worst:.2e}")
