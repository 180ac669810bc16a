"""GPU parity for the multi-model pool (the paper's "All" experiment).

Several fitted models of ranks R_m are jackknifed at once: all their submodels share one fused
multi-factor per mode with per-model block widths (CALS's sum_i R_i, PAPER.md:291-292;
SPEC.md:234-239). The pool changes only the arrangement of the work, so the oracle is the
plain per-model delete-d JK-ALS (orc_jk_als_d), run once per model; the bar is the same as
for a single model (factors within 1e-10 relative, errors 1e-9 rel + 1e-13 ||T_-g||^2).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_pool

pytestmark = pytest.mark.gpu

FTOL = 1e-10
NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def run_pool(w, sweeps, d=1, tol=0.0, sub_range=None, precision=0):
    from paper_2112_03985_b200 import JKCals
    h = JKCals(w.T, list(w.ranks), sub_range=sub_range, hist_cap=max(sweeps, 1), d=d, precision=precision)
    h.set_init(w.Ps)
    done = h.iterate(sweeps, tol)
    return h, done


def oracle_pool(w, sweeps, d=1, tol=0.0, subs=None):
    """{submodel id: (JKResult, q)} from per-model oracle runs over the requested ids."""
    G = -(-w.dims[0] // d)
    subs = list(range(len(w.ranks) * G)) if subs is None else list(subs)
    out = {}
    for m, P in enumerate(w.Ps):
        gl = [s % G for s in subs if s // G == m]
        if not gl:
            continue
        res = O.jk_als_d(w.T, P, d, g_list=gl, max_iters=sweeps, tol=tol, nthreads=NCPU)
        for q, g in enumerate(gl):
            out[m * G + g] = (res, q)
    return out


def check(h, orc, w, d, ftol=FTOL, etol=1e-9, hist=True):
    G = -(-w.dims[0] // d)
    s_all = O.slice_norms_sq(w.T, 0)
    n2 = O.norm_sq(w.T)
    st = h.status()
    for s, (res, q) in orc.items():
        m, g = divmod(s, G)
        rows = list(range(g * d, min(g * d + d, w.dims[0])))
        fac, lam = h.factors(s)
        assert fac[1].shape == (w.dims[1], w.ranks[m])
        for n, (a, b) in enumerate(zip(fac, res.factors[q])):
            assert rel(a, b) <= ftol, (s, n, rel(a, b))
        assert rel(lam, res.lam[q]) <= ftol, (s, rel(lam, res.lam[q]))
        if hist:
            hg, ho = h.history(s), res.history(q)
            assert len(hg) == len(ho) == res.iters[q]
            nt2 = n2 - s_all[rows].sum()
            assert np.all(np.abs(hg - ho) <= etol * np.abs(ho) + 1e-13 * nt2), (s, np.abs(hg - ho).max())
        assert st["iters"][s - h.sub_begin] == res.iters[q]
        assert np.all(h.block(s, 0)[rows] == 0.0)


def test_pool_mixed_ranks_all_submodels():
    w = make_pool(((30, 20, 12), (2, 3, 5), 5, 0.01, "syn", 40), seed=3)
    h, _ = run_pool(w, 40)
    assert h.nsub == 90
    check(h, oracle_pool(w, 40), w, 1)


def test_pool_equal_ranks_two_models():
    # two models of the same rank: the uniform-width fast path with two warm starts
    w = make_pool(((20, 15, 10), (3, 3), 4, 0.01, "syn", 30), seed=8)
    h, _ = run_pool(w, 30)
    check(h, oracle_pool(w, 30), w, 1)


def test_pool_delete_d_shard_across_models():
    # delete-d (d = 4, I_0 = 30: 8 groups, last of 2) with a shard [5, 19) crossing the model
    # boundaries 8 and 16 of a 3-model pool
    w = make_pool(((30, 20, 12), (4, 2, 5), 5, 0.01, "syn", 30), seed=5)
    h, _ = run_pool(w, 30, d=4, sub_range=(5, 19))
    orc = oracle_pool(w, 30, d=4, subs=range(5, 19))
    check(h, orc, w, 4)
    # all_factors: packed per submodel with per-model ranks and per-group rows
    U0, lam = h.all_factors(0)
    U2, _ = h.all_factors(2)
    for q, s in enumerate(range(5, 19)):
        fac, lg = h.factors(s)
        assert np.array_equal(U0[q], fac[0]) and np.array_equal(U2[q], fac[2])
        assert np.array_equal(lam[q], lg)


def test_pool_paper_all_small_sampled():
    # the paper's "All" pool: 50 x 100 x 100, R in {3, 5, 7, 9}, 20 sweeps,
    # sampled submodels of every model (R = 7, 9 over-factor the rank-5 truth: DESIGN.md A17)
    w = make_pool("all_small", sweeps=20)
    h, _ = run_pool(w, 20)
    G = 50
    subs = [m * G + g for m in range(4) for g in (0, 1, 25, 49)]
    orc = oracle_pool(w, 20, subs=subs)
    check(h, orc, w, 1)


def test_pool_tolerance_compaction_mixed():
    # tol > 0: submodels of different widths converge at different sweeps and are compacted out
    w = make_pool(((24, 16, 10), (2, 4, 3), 4, 0.01, "syn", 300), seed=11)
    h, done = run_pool(w, 300, tol=1e-8)
    orc = oracle_pool(w, 300, tol=1e-8)
    assert done == max(res.iters[q] for res, q in orc.values())
    check(h, orc, w, 1)


def test_pool_stats_per_model():
    w = make_pool(((20, 15, 10), (2, 3), 3, 0.01, "syn", 25), seed=2)
    h, _ = run_pool(w, 25)
    for m, R in enumerate(w.ranks):
        res = O.jk_als(w.T, w.Ps[m], max_iters=25, nthreads=NCPU)
        for mode in (1, 2):
            mean, std = h.jackknife_stats(mode, model=m)
            om, os_ = O.jackknife_stats(np.stack([f[mode] for f in res.factors]))
            assert mean.shape == (w.dims[mode], R)
            assert rel(mean, om) <= 1e-10 and rel(std, os_) <= 1e-8


def test_pool_fp32_path():
    w = make_pool(((40, 30, 20), (2, 4, 3), 4, 0.01, "syn", 30), seed=6)
    h, _ = run_pool(w, 30, precision=1)
    orc = oracle_pool(w, 30)
    for s, (res, q) in orc.items():
        fac, _ = h.factors(s)
        for a, b in zip(fac, res.factors[q]):
            assert rel(a, b) <= 1e-4, (s, rel(a, b))
