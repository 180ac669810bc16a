"""GPU parity for submodel alignment and the aligned ("full") jackknife statistics (NEXT #3).

Alg. 2 alg:jk:perm_scale + alg:jk:std with the scheme of DESIGN.md
reading A12 / A20. The oracle aligns its own JK-ALS submodels (orc_align) to the same warm start;
permutations and signs must match exactly, aligned factors within 1e-10 relative.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_pool, make_workload

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def groups_of(I0, d):
    return [list(range(g * d, min(g * d + d, I0))) for g in range(-(-I0 // d))]


def check_aligned(h, w, res, P, subs, groups, ftol=1e-10):
    """res.factors[q] is the oracle submodel of h's submodel subs[q]; returns the oracle's
    aligned factors per q."""
    out = []
    for q, s in enumerate(subs):
        al, perm, sign, cong = O.align(res.factors[q], res.lam[q], P)
        gp, gs, gc = h.alignment(s)
        assert np.array_equal(gp, perm), (s, gp, perm)
        assert np.array_equal(gs, sign), (s, gs, sign)
        assert np.allclose(gc, cong, rtol=1e-12, atol=1e-14)
        ga = h.aligned_factors(s)
        for n, (a, b) in enumerate(zip(ga, al)):
            assert rel(a, b) <= ftol, (s, n, rel(a, b))
        out.append(al)
    return out


def test_align_tiny_and_full_stats():
    from paper_2112_03985_b200 import JKCals
    w = make_workload("tiny")
    h = JKCals(w.T, w.R, hist_cap=w.sweeps)
    h.set_init(w.P)
    h.iterate(w.sweeps, 0.0)
    h.align()
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    al = check_aligned(h, w, res, w.P, range(10), groups_of(10, 1))
    # full stats: modes >= 1 over all submodels, mode 0 over the submodels containing the row
    for mode in range(3):
        if mode == 0:
            X = np.stack([O.mode0_full(al[q][0], [q], 10) for q in range(10)])
        else:
            X = np.stack([al[q][mode] for q in range(10)])
        om, os_, oc = O.present_stats(X)
        cnt, mean, m2 = h.aligned_moments(mode)
        gm, gs = h.aligned_stats(mode)
        assert np.array_equal(cnt, oc)
        assert rel(gm, om) <= 1e-10 and rel(gs, os_) <= 1e-8, (mode, rel(gm, om), rel(gs, os_))


def test_align_pool_delete_d_mixed():
    from paper_2112_03985_b200 import JKCals
    w = make_pool(((21, 14, 9), (2, 4, 3), 4, 0.01, "syn", 30), seed=4)
    d, G = 3, 7
    h = JKCals(w.T, list(w.ranks), hist_cap=30, d=d)
    h.set_init(w.Ps)
    h.iterate(30, 0.0)
    h.align()
    for m, P in enumerate(w.Ps):
        res = O.jk_als_d(w.T, P, d, max_iters=30, nthreads=NCPU)
        subs = [m * G + g for g in range(G)]
        al = check_aligned(h, w, res, P, subs, groups_of(21, d))
        for mode in range(3):
            if mode == 0:
                X = np.stack([O.mode0_full(al[g][0], groups_of(21, d)[g], 21) for g in range(G)])
            else:
                X = np.stack([al[g][mode] for g in range(G)])
            om, os_, oc = O.present_stats(X)
            cnt, mean, _ = h.aligned_moments(mode, model=m)
            gm, gs = h.aligned_stats(mode, model=m)
            assert np.array_equal(cnt, oc)
            assert rel(gm, om) <= 1e-10 and rel(gs, os_) <= 1e-8


def test_align_recovers_injected_permutation_and_signs():
    # permute and negate submodel columns through set_init_submodel: the alignment undoes it
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r4")
    h = JKCals(w.T, w.R, hist_cap=20)
    h.set_init(w.P)
    h.iterate(20, 0.0)
    pi = np.array([2, 3, 0, 1])
    for p in (0, 17, 49):
        fac, _ = h.factors(p)
        for n in range(3):
            f = fac[n][:, pi].copy()
            if n == 1:
                f[:, 0] *= -1
            if n == 2:
                f[:, 0] *= -1
            h.set_init_submodel(p, n, f)
    h.align()
    for p in (0, 17, 49):
        perm, sign, _ = h.alignment(p)
        assert np.array_equal(perm, pi)          # column r came from reference column pi[r]
        assert sign[1, 0] == -1 and sign[2, 0] == -1 and sign[0, 0] == 1
    perm, sign, _ = h.alignment(5)
    assert np.array_equal(perm, np.arange(4)) and np.all(sign == 1)


def test_align_state_and_rank_errors():
    from paper_2112_03985_b200 import JKCals, JKCalsError
    w = make_workload("tiny")
    h = JKCals(w.T, w.R, hist_cap=5)
    h.set_init(w.P)
    h.iterate(5, 0.0)
    with pytest.raises(JKCalsError):
        h.aligned_factors(0)                      # E_STATE: not aligned yet
    h.align()
    h.aligned_factors(0)
    h.iterate(1, 0.0)
    with pytest.raises(JKCalsError):
        h.alignment(0)                            # stale after iterate
    g = np.random.default_rng(0)
    T = g.standard_normal((4, 12, 12))
    h2 = JKCals(T, 11, hist_cap=2)
    h2.set_init([g.standard_normal((I, 11)) for I in (4, 12, 12)])
    with pytest.raises(JKCalsError):
        h2.align()                                # E_SHAPE: rank > 10
