"""GPU parity for plain CALS (§3.3): K CP models of one
tensor fitted concurrently by one fused sweep (no left-out rows). Oracle: independent
orc_cp_als per model from the same initial model (CALS "does not alter the numerics" of ALS,
PAPER.md:111). Bar: factors within 1e-10 relative, error histories 1e-9 relative."""
import numpy as np
import pytest

from oracle import oracle as O
from synth import make_workload

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def random_inits(dims, ranks, seed):
    g = np.random.default_rng(seed)
    return [[np.asfortranarray(g.uniform(0, 1, (I, R))) for I in dims] for R in ranks]


def check(h, T, inits, sweeps, tol=0.0, ftol=1e-10):
    st = h.status()
    for m, U0 in enumerate(inits):
        U, lam, hist, iters, flags = O.cp_als(T, U0, sweeps, tol)
        fac, gl = h.factors(m)
        assert fac[0].shape == U[0].shape          # nothing left out
        for n, (a, b) in enumerate(zip(fac, U)):
            assert rel(a, b) <= ftol, (m, n, rel(a, b))
        assert rel(gl, lam) <= ftol
        hg = h.history(m)
        assert len(hg) == iters == st["iters"][m]
        assert np.allclose(hg, hist, rtol=1e-9, atol=1e-13 * O.norm_sq(T))


def test_cals_multistart_same_rank():
    # the paper's CALS use case: many random starts of one rank
    from paper_2112_03985_b200 import cals
    w = make_workload("syn50_r3")
    inits = random_inits(w.dims, [3] * 20, seed=1)
    h = cals(w.T, [3] * 20, inits, hist_cap=40)
    h.iterate(40, 0.0)
    check(h, w.T, inits, 40)


def test_cals_mixed_ranks_tolerance():
    # models of ranks 1..6, tol > 0: each stops on its own and is compacted out
    from paper_2112_03985_b200 import cals
    w = make_workload(((30, 20, 10), 4, 4, 0.01, "syn", 300), seed=2)
    ranks = [1, 2, 3, 4, 5, 6, 2, 4]
    inits = random_inits(w.dims, ranks, seed=3)
    h = cals(w.T, ranks, inits, hist_cap=300)
    h.iterate(300, 1e-7)
    check(h, w.T, inits, 300, tol=1e-7, ftol=1e-9)


def test_cals_fp32_and_4way():
    from paper_2112_03985_b200 import cals
    w = make_workload(((20, 12, 10, 8), 3, 3, 0.01, "syn", 30), seed=4)
    inits = random_inits(w.dims, [3, 3, 2], seed=5)
    h = cals(w.T, [3, 3, 2], inits, hist_cap=30)
    h.iterate(30, 0.0)
    check(h, w.T, inits, 30)
    h32 = cals(w.T, [3, 3, 2], inits, hist_cap=30, precision=1)
    h32.iterate(30, 0.0)
    for m, U0 in enumerate(inits):
        U, *_ = O.cp_als(w.T, U0, 30)
        for a, b in zip(h32.factors(m)[0], U):
            assert rel(a, b) <= 1e-4
