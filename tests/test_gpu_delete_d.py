"""GPU parity for delete-d jackknife ("pad and periodically zero out d rows").

Group g leaves out mode-0 rows [g d, min(g d + d, I_0)) (last group smaller).
The CUDA path (C ABI jkcals_create_d) is compared with the oracle's delete-d JK-ALS
(orc_jk_als_d, which physically removes the group's slices) at the same bar as leave-one-out:
factors within 1e-10 relative Frobenius, per-sweep errors within 1e-9 rel + 1e-13 ||T_-g||^2.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_workload

pytestmark = pytest.mark.gpu

FTOL = 1e-10
NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def run_gpu(w, d, sweeps, tol=0.0, sub_range=None, precision=0):
    from paper_2112_03985_b200 import JKCals
    h = JKCals(w.T, w.R, sub_range=sub_range, hist_cap=max(sweeps, 1), d=d, precision=precision)
    h.set_init(w.P)
    done = h.iterate(sweeps, tol)
    return h, done


def nt2g_of(T, d):
    s = O.slice_norms_sq(T, 0)
    return np.array([O.norm_sq(T) - s[g].sum() for g in O.delete_d_groups(T.shape[0], d)])


def check(h, res, groups, d, T, ftol=FTOL, etol=1e-9):
    st = h.status()
    nt2g = nt2g_of(T, d)
    for q, g in enumerate(groups):
        rows = O.delete_d_groups(T.shape[0], d)[g]
        fac, lam = h.factors(g)
        assert fac[0].shape == (T.shape[0] - len(rows), w_R(res))
        for n, (a, b) in enumerate(zip(fac, res.factors[q])):
            assert rel(a, b) <= ftol, (g, n, rel(a, b))
        assert rel(lam, res.lam[q]) <= ftol
        hg, ho = h.history(g), res.history(q)
        assert len(hg) == len(ho) == res.iters[q]
        assert np.all(np.abs(hg - ho) <= etol * np.abs(ho) + 1e-13 * nt2g[g]), (g, np.abs(hg - ho).max())
        sub = g - h.sub_begin
        assert st["iters"][sub] == res.iters[q]
        # padded-row invariant for d rows: the group's rows are bitwise zero
        blk = h.block(g, 0)
        assert np.all(blk[rows] == 0.0)


def w_R(res):
    return res.R


@pytest.mark.parametrize("d", [2, 3, 5])
def test_tiny_delete_d_all_groups(d):
    # I_0 = 10: d = 3 leaves a ragged last group of one row
    w = make_workload("tiny")
    h, done = run_gpu(w, d, w.sweeps)
    assert done == w.sweeps
    res = O.jk_als_d(w.T, w.P, d, max_iters=w.sweeps, nthreads=NCPU)
    G = range(-(-10 // d))
    assert h.nsub == len(G)
    check(h, res, G, d, w.T)


@pytest.mark.parametrize("d", [4, 25])
def test_syn50_delete_d(d):
    # d = 25 = I_0/2 is the largest d the paper allows; d = 4 is ragged (50 = 12*4 + 2)
    w = make_workload("syn50_r3")
    h, _ = run_gpu(w, d, w.sweeps)
    res = O.jk_als_d(w.T, w.P, d, max_iters=w.sweeps, nthreads=NCPU)
    check(h, res, range(-(-50 // d)), d, w.T)


def test_delete_d_all_factors_ragged_and_shard():
    # a shard [1, 4) of the 4 groups of I_0 = 10, d = 3 (the last group, rows {9}, is ragged);
    # all_factors must agree with per-group factors
    w = make_workload("tiny")
    h, _ = run_gpu(w, 3, 20, sub_range=(1, 4))
    res = O.jk_als_d(w.T, w.P, 3, g_list=[1, 2, 3], max_iters=20, nthreads=NCPU)
    check(h, res, [1, 2, 3], 3, w.T)
    U0, lam = h.all_factors(0)
    assert isinstance(U0, list) and [u.shape[0] for u in U0] == [7, 7, 9]
    for q, g in enumerate([1, 2, 3]):
        fac, lg = h.factors(g)
        assert np.array_equal(U0[q], fac[0]) and np.array_equal(lam[q], lg)
    U1, _ = h.all_factors(1)
    for q, g in enumerate([1, 2, 3]):
        assert np.array_equal(U1[q], h.factors(g)[0][1])


def test_delete_d1_is_leave_one_out_bitwise():
    # d = 1 through jkcals_create_d is the leave-one-out path, bit for bit
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r2")
    a = JKCals(w.T, w.R, hist_cap=30)
    a.set_init(w.P)
    a.iterate(30, 0.0)
    b = JKCals(w.T, w.R, hist_cap=30, d=1)
    b.set_init(w.P)
    b.iterate(30, 0.0)
    for n in range(3):
        assert np.array_equal(a.all_factors(n)[0], b.all_factors(n)[0])


def test_delete_d_tolerance_and_compaction():
    # tol > 0: groups converge independently and are compacted out; results still match the oracle
    w = make_workload("syn50_r4")
    d = 4
    h, done = run_gpu(w, d, 200, tol=1e-9)
    res = O.jk_als_d(w.T, w.P, d, max_iters=200, tol=1e-9, nthreads=NCPU)
    assert done == res.iters.max()
    check(h, res, range(13), d, w.T)


def test_delete_d_fp32_path():
    # the 3xTF32 tcgen05 path with padded groups, at the FP32 bar (1e-4)
    w = make_workload("syn50_r5")
    h, _ = run_gpu(w, 5, w.sweeps, precision=1)
    res = O.jk_als_d(w.T, w.P, 5, max_iters=w.sweeps, nthreads=NCPU)
    for g in range(10):
        fac, _ = h.factors(g)
        for a, b in zip(fac, res.factors[g]):
            assert rel(a, b) <= 1e-4, (g, rel(a, b))
        assert np.all(h.block(g, 0)[g * 5:g * 5 + 5] == 0.0)


def test_delete_d_set_init_submodel_roundtrip():
    # set_init_submodel takes the get_factors layout ((I_0 - |group|) x R for mode 0)
    w = make_workload("tiny")
    h, _ = run_gpu(w, 3, 10)
    fac, _ = h.factors(3)          # ragged group {9}
    h.set_init_submodel(3, 0, fac[0] * 2.0)
    blk = h.block(3, 0)
    assert np.array_equal(blk[:9], fac[0] * 2.0) and np.all(blk[9] == 0.0)
    fac1, _ = h.factors(1)         # group {3, 4, 5}
    h.set_init_submodel(1, 0, fac1[0])
    blk = h.block(1, 0)
    assert np.all(blk[3:6] == 0.0) and np.array_equal(np.delete(blk, [3, 4, 5], axis=0), fac1[0])


def test_delete_d_rejects_bad_d():
    from paper_2112_03985_b200 import JKCals, JKCalsError
    w = make_workload("tiny")
    for d, rng_ in [(-1, None), (6, None), (3, (0, 5))]:   # (d = 0 is plain CALS)
        with pytest.raises(JKCalsError):
            JKCals(w.T, w.R, d=d, sub_range=rng_)
