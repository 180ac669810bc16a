"""GPU parity of the cluster-resident whole-iterate path (csrc/resident.cuh) for small tensors.

One launch runs every sweep: T split along its last mode over the CTAs of a thread-block
cluster (shared memory), factor replicas per CTA, DSMEM gathers of the partial MTTKRP blocks,
per-submodel ALS updates by owner CTAs (Alg. 3). Held to the same bar as the
standard path: factors within 1e-10 relative Frobenius of the oracle's JK-ALS, per-sweep errors
within 1e-9 rel + 1e-13 ||T_-p||^2, iteration counts and flags exact, padded rows bitwise zero.
JKCALS_RESIDENT=1 forces the path wherever it fits, =0 disables it (read at each iterate).
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


@pytest.fixture
def resident(monkeypatch):
    monkeypatch.setenv("JKCALS_RESIDENT", "1")


def fit(T, P, R, sweeps, tol=0.0, d=1, hist=None, instrument=False):
    from paper_2112_03985_b200 import JKCals
    h = JKCals(T, R, hist_cap=hist or max(sweeps, 1), d=d)
    h.set_init(P)
    if instrument:
        h.set_instrument(True)
    done = h.iterate(sweeps, tol)
    return h, done


def check(h, res, ids, T, d=1):
    s = O.slice_norms_sq(T, 0)
    n2 = O.norm_sq(T)
    groups = O.delete_d_groups(T.shape[0], d)
    st = h.status()
    for q, p in enumerate(ids):
        fac, lam = h.factors(p)
        for n, (a, b) in enumerate(zip(fac, res.factors[q])):
            assert rel(a, b) <= FTOL, (p, n, rel(a, b))
        assert rel(lam, res.lam[q]) <= FTOL, (p, rel(lam, res.lam[q]))
        hg, ho = h.history(p), res.history(q)
        assert len(hg) == len(ho) == res.iters[q]
        nt2 = n2 - s[groups[p]].sum()
        assert np.all(np.abs(hg - ho) <= 1e-9 * np.abs(ho) + 1e-13 * nt2), (p, np.abs(hg - ho).max())
        assert st["iters"][p] == res.iters[q]
        assert (st["flags"][p] & ~1) == (res.flags[q] & ~1)
        assert np.all(h.block(p, 0)[groups[p]] == 0.0)


@pytest.mark.parametrize("name", ["tiny", "syn50_r1", "syn50_r3", "syn50_r5"])
def test_resident_all_submodels_vs_oracle(resident, name):
    w = make_workload(name)
    h, done = fit(w.T, w.P, w.R, w.sweeps, instrument=True)
    assert done == w.sweeps
    tm, te, nl = h.kernel_times()
    assert nl == 1  # the whole iterate was one (cluster-resident) launch
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    check(h, res, range(w.dims[0]), w.T)


def test_resident_deterministic(resident):
    w = make_workload("syn50_r2")
    h1, _ = fit(w.T, w.P, w.R, 15)
    h2, _ = fit(w.T, w.P, w.R, 15)
    for p in (0, 17, 49):
        for a, b in zip(h1.factors(p)[0], h2.factors(p)[0]):
            assert np.array_equal(a, b)


def test_resident_tol_mode_device_stop(resident):
    w = make_workload("syn50_r3")
    h, done = fit(w.T, w.P, w.R, 1000, tol=1e-6, hist=1000)
    res = O.jk_als(w.T, w.P, max_iters=1000, tol=1e-6, nthreads=NCPU)
    assert len(set(res.iters.tolist())) > 1
    assert done == res.iters.max()
    check(h, res, range(50), w.T)


@pytest.mark.parametrize("dims,R,d", [((12, 9, 7, 5), 3, 1), ((9, 11, 6), 2, 2), ((7, 5, 6, 4, 3), 2, 1),
                                      ((25, 13, 17), 7, 3)])
def test_resident_shapes_and_delete_d(resident, dims, R, d):
    g = np.random.default_rng(sum(dims) + R)
    A = [g.uniform(0, 1, (I, R)) for I in dims]
    T = np.zeros(dims)  # planted CP tensor, any N
    for r in range(R):
        t = A[0][:, r]
        for a in A[1:]:
            t = np.multiply.outer(t, a[:, r])
        T += t
    T = np.asfortranarray(T + 0.01 * g.standard_normal(dims))
    P = [np.asfortranarray(a + 0.05 * g.standard_normal(a.shape)) for a in A]
    sweeps = 30
    h, _ = fit(T, P, R, sweeps, d=d)
    if d == 1:
        res = O.jk_als(T, P, max_iters=sweeps, nthreads=NCPU)
    else:
        res = O.jk_als_d(T, P, d, max_iters=sweeps, nthreads=NCPU)
    check(h, res, range(len(O.delete_d_groups(dims[0], d))), T, d=d)


def test_resident_and_standard_paths_continue_each_other(monkeypatch):
    """State written back by the resident launch continues on the standard path: 20 resident
    sweeps, the factors carried into a second handle, 20 standard sweeps == 40 oracle sweeps."""
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r2")
    monkeypatch.setenv("JKCALS_RESIDENT", "1")
    h = JKCals(w.T, w.R, hist_cap=60)
    h.set_init(w.P)
    h.iterate(20, 0.0)
    monkeypatch.setenv("JKCALS_RESIDENT", "0")
    h2 = JKCals(w.T, w.R, hist_cap=60)
    h2.set_init(w.P)
    for m in range(3):
        U, _ = h.all_factors(m)
        h2.set_init_all(m, U)
    h2.set_instrument(True)
    h2.iterate(20, 0.0)
    assert h2.kernel_times()[2] == 20 * 3  # the standard path: per-mode launches
    res = O.jk_als(w.T, w.P, max_iters=40, nthreads=NCPU)
    for p in range(50):
        fac, _ = h2.factors(p)
        for a, b in zip(fac, res.factors[p]):
            assert rel(a, b) <= 1e-9, (p, rel(a, b))


# ---------------------------------------------------------------- warp-per-submodel kernel (tiny)
@pytest.fixture
def warp_path(monkeypatch):
    monkeypatch.setenv("JKCALS_RESIDENT", "2")


def _planted(dims, R, seed):
    g = np.random.default_rng(seed)
    A = [g.uniform(0, 1, (I, R)) for I in dims]
    T = np.zeros(dims)
    for r in range(R):
        t = A[0][:, r]
        for a_ in A[1:]:
            t = np.multiply.outer(t, a_[:, r])
        T += t
    T = np.asfortranarray(T + 0.01 * g.standard_normal(dims))
    P = [np.asfortranarray(a_ + 0.05 * g.standard_normal(a_.shape)) for a_ in A]
    return T, P


def test_warp_tiny_all_submodels(warp_path):
    w = make_workload("tiny")
    h, done = fit(w.T, w.P, w.R, w.sweeps, instrument=True)
    assert done == w.sweeps and h.kernel_times()[2] == 1
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    check(h, res, range(w.dims[0]), w.T)


@pytest.mark.parametrize("dims,R,d,tol", [((12, 9, 7), 3, 1, 0.0), ((7, 5, 6, 4), 2, 1, 0.0), ((9, 6, 5), 4, 2, 0.0),
                                          ((11, 8, 6), 2, 1, 1e-6), ((6, 5, 4, 3, 2), 3, 1, 0.0)])
def test_warp_shapes_delete_d_tol(warp_path, dims, R, d, tol):
    T, P = _planted(dims, R, sum(dims) + R)
    sweeps = 200 if tol > 0 else 40
    h, done = fit(T, P, R, sweeps, tol=tol, d=d, hist=sweeps)
    if d == 1:
        res = O.jk_als(T, P, max_iters=sweeps, tol=tol, nthreads=NCPU)
    else:
        res = O.jk_als_d(T, P, d, max_iters=sweeps, tol=tol, nthreads=NCPU)
    if tol > 0:
        assert done == res.iters.max()
    check(h, res, range(len(O.delete_d_groups(dims[0], d))), T, d=d)
