"""GPU robustness tests from SURVEY §4 / §5 (SPEC acceptance items): fusion transparency,
the padded-row invariant after EVERY sweep, monotone error histories, per-submodel fault
isolation, and checkpoint / resume through get_factors + set_init_submodel."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_workload

pytestmark = pytest.mark.gpu
NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def test_fusion_transparency_block_equals_solo():
    # a submodel fitted inside the fused batch equals the same submodel
    # fitted alone (only the split-K summation order differs: rounding level)
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r3")
    full = JKCals(w.T, w.R, hist_cap=100)
    full.set_init(w.P)
    full.iterate(100, 0.0)
    for p in (0, 17, 49):
        solo = JKCals(w.T, w.R, sub_range=(p, p + 1), hist_cap=100)
        solo.set_init(w.P)
        solo.iterate(100, 0.0)
        fa, la = full.factors(p)
        fb, lb = solo.factors(p)
        for a, b in zip(fa, fb):
            assert rel(a, b) <= 1e-12, (p, rel(a, b))
        assert np.allclose(full.history(p), solo.history(p), rtol=1e-12)


@pytest.mark.parametrize("d", [1, 3])
def test_padded_rows_zero_after_every_sweep(d):
    # the group's rows are bitwise zero in the fused mode-0 factor after
    # every sweep (checked sweep by sweep, graph replay path)
    from paper_2112_03985_b200 import JKCals
    w = make_workload("tiny")
    h = JKCals(w.T, w.R, hist_cap=20, d=d)
    h.set_init(w.P)
    G = -(-10 // d)
    for sweep in range(20):
        h.iterate(1, 0.0)
        for g in range(G):
            rows = list(range(g * d, min(g * d + d, 10)))
            assert np.all(h.block(g, 0)[rows] == 0.0), (sweep, g)


def test_error_history_monotone():
    # ALS never increases the error (slack 1e-12 ||T||^2) -- on the GPU histories
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r4")
    h = JKCals(w.T, w.R, hist_cap=100)
    h.set_init(w.P)
    h.iterate(100, 0.0)
    slack = 1e-12 * O.norm_sq(w.T)
    for p in range(50):
        e = h.history(p)
        assert np.all(np.diff(e) <= slack), (p, np.diff(e).max())


@pytest.mark.parametrize("prec", [0, 2])  # FP64 DMMA, FP64_I8 (per-column U exponents + NaN marker)
def test_fault_isolated_to_one_submodel(prec):
    # SURVEY §5 fault injection: a submodel driven to overflow (factor scaled by 1e300) is
    # flagged non-finite and frozen; every other submodel is untouched (vs a clean run)
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r2")
    clean = JKCals(w.T, w.R, hist_cap=30, precision=prec)
    clean.set_init(w.P)
    clean.iterate(30, 0.0)
    h = JKCals(w.T, w.R, hist_cap=30, precision=prec)
    h.set_init(w.P)
    bad = w.P[2] * 1e300
    h.set_init_submodel(7, 2, bad)
    h.set_init_submodel(7, 1, w.P[1] * 1e300)
    h.iterate(30, 0.0)
    st = h.status()
    assert st["flags"][7] & 4, st["flags"][7]            # F_NONFINITE
    assert st["iters"][7] < 30                             # frozen
    for p in range(50):
        if p == 7:
            continue
        assert not (st["flags"][p] & 4)
        for a, b in zip(h.factors(p)[0], clean.factors(p)[0]):
            assert rel(a, b) <= 1e-12


def test_checkpoint_resume():
    # get_factors + set_init_submodel resume. 20 sweeps, checkpoint every submodel,
    # resume in a fresh handle for 20 more == 40 sweeps straight (oracle at 1e-10)
    from paper_2112_03985_b200 import JKCals
    w = make_workload("tiny")
    a = JKCals(w.T, w.R, hist_cap=40)
    a.set_init(w.P)
    a.iterate(20, 0.0)
    ck = {p: a.factors(p)[0] for p in range(10)}
    b = JKCals(w.T, w.R, hist_cap=40)
    b.set_init(w.P)
    for p, fac in ck.items():
        for n, U in enumerate(fac):
            b.set_init_submodel(p, n, U)
    b.iterate(20, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=40, nthreads=NCPU)
    for p in range(10):
        for x, y in zip(b.factors(p)[0], res.factors[p]):
            assert rel(x, y) <= 1e-10, (p, rel(x, y))


def test_c_abi_from_plain_c(tmp_path):
    # the boundary is a C ABI: a plain C99 program (tests/c_abi_demo.c, gcc, no Python) drives
    # create / set_init / iterate / get_factors and must produce exactly the binding's results
    import subprocess
    from paper_2112_03985_b200 import JKCals, _build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(_build.LIB)
    exe = tmp_path / "c_abi_demo"
    subprocess.check_call(["gcc", "-std=c99", "-O2", os.path.join(root, "tests", "c_abi_demo.c"),
                           "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                           "-L", libdir, "-ljkcals", "-L", "/usr/local/cuda/lib64", "-lcudart",
                           "-Wl,-rpath," + libdir, "-o", str(exe)])
    w = make_workload("tiny")
    sweeps = 20
    with open(tmp_path / "in.bin", "wb") as f:
        np.array([len(w.dims), *w.dims, w.R], dtype=np.int64).tofile(f)
        np.ravel(w.T, order="F").tofile(f)
        for p in w.P:
            np.ravel(p, order="F").tofile(f)
    out = subprocess.run([str(exe), str(tmp_path / "in.bin"), str(tmp_path / "out.bin"), str(sweeps)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    got = np.fromfile(tmp_path / "out.bin")
    h = JKCals(w.T, w.R, hist_cap=sweeps)
    h.set_init(w.P)
    h.iterate(sweeps, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=sweeps, nthreads=NCPU)
    off = 0
    for p in range(10):
        fac, lam = h.factors(p)
        for n, U in enumerate(fac):
            blk = got[off:off + U.size].reshape(U.shape, order="F")
            off += U.size
            assert np.array_equal(blk, U), (p, n)          # same library, same results, bitwise
            assert rel(blk, res.factors[p][n]) <= 1e-10
        assert np.array_equal(got[off:off + w.R], lam)
        off += w.R
    assert off == got.size


def test_checkpoint_resume_all_factors_pool():
    # batched resume: all_factors per mode -> set_init_all on a fresh handle (a mixed-rank pool
    # with a ragged delete-d group), then the continued fit equals one straight run
    from paper_2112_03985_b200 import JKCals
    from synth import make_pool
    w = make_pool(((11, 7, 6), (2, 3), 3, 0.01, "syn", 20), seed=3)
    a = JKCals(w.T, list(w.ranks), hist_cap=30, d=3)
    a.set_init(w.Ps)
    a.iterate(12, 0.0)
    ck = [a.all_factors(n)[0] for n in range(3)]
    b = JKCals(w.T, list(w.ranks), hist_cap=30, d=3)
    b.set_init(w.Ps)
    for n in range(3):
        b.set_init_all(n, ck[n])
    for n in range(3):
        got = b.all_factors(n)[0]
        for x, y in zip(got, ck[n]):
            assert np.array_equal(x, y)
    b.iterate(18, 0.0)
    for m, P in enumerate(w.Ps):
        res = O.jk_als_d(w.T, P, 3, max_iters=30, nthreads=NCPU)
        for g in range(4):
            for x, y in zip(b.factors(m * 4 + g)[0], res.factors[g]):
                assert rel(x, y) <= 1e-10


@pytest.mark.parametrize("R", [7, 10, 12, 16])
def test_large_ranks_epilogue_classes(R):
    # the R > 8 rank classes (RMAX 10 / 12 / 16 epilogues, 16 = the ABI maximum) vs the oracle
    from paper_2112_03985_b200 import JKCals
    w = make_workload(((12, 30, 28), R, 16, 0.01, "syn", 15), seed=R)
    h = JKCals(w.T, w.R, hist_cap=15)
    h.set_init(w.P)
    h.iterate(15, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=15, nthreads=NCPU)
    for p in (0, 5, 11):
        for a, b in zip(h.factors(p)[0], res.factors[p]):
            assert rel(a, b) <= 1e-10, (R, p, rel(a, b))


@pytest.mark.parametrize("R", [17, 20, 32])
def test_ranks_above_16_streaming_epilogue(R):
    # ranks 17..32 run the streaming large-rank epilogue (epilogue_large.cuh); I_1 = 300 > one
    # 128-row chunk, I_0 = 9 submodels
    from paper_2112_03985_b200 import JKCals
    w = make_workload(((9, 300, 40), R, 32, 0.01, "syn", 12), seed=R)
    h = JKCals(w.T, w.R, hist_cap=12)
    h.set_init(w.P)
    h.iterate(12, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=12, nthreads=NCPU)
    for p in range(9):
        fac, lam = h.factors(p)
        for a, b in zip(fac, res.factors[p]):
            assert rel(a, b) <= 1e-10, (R, p, rel(a, b))
        assert rel(lam, res.lam[p]) <= 1e-10
        assert np.allclose(h.history(p), res.history(p), rtol=1e-9, atol=1e-13 * O.norm_sq(w.T))


def test_paper_application_pool_ranks_19_20_21():
    # the paper's second application jackknifes three models of ranks {19, 20, 21} together
    # (PAPER.md:590-596); here on a small 44 x 120 x 30 tensor with delete-2 groups
    from paper_2112_03985_b200 import JKCals
    from synth import make_pool
    w = make_pool(((44, 120, 30), (19, 20, 21), 20, 0.01, "syn", 8), seed=5)
    h = JKCals(w.T, list(w.ranks), hist_cap=8, d=2)
    h.set_init(w.Ps)
    h.iterate(8, 0.0)
    for m, P in enumerate(w.Ps):
        res = O.jk_als_d(w.T, P, 2, g_list=[0, 21], max_iters=8, nthreads=NCPU)
        for q, g in enumerate([0, 21]):
            fac, _ = h.factors(m * 22 + g)
            for a, b in zip(fac, res.factors[q]):
                assert rel(a, b) <= 1e-10, (m, g, rel(a, b))


def test_large_rank_pinv_fallback():
    # the large-rank epilogue's Jacobi pseudoinverse (shared-memory scratch): a zero column in
    # one submodel's mode-1 init makes its H singular; it matches the oracle's pinv path
    from paper_2112_03985_b200 import JKCals
    w = make_workload(((8, 60, 40), 18, 32, 0.01, "syn", 10), seed=18)
    h = JKCals(w.T, w.R, hist_cap=10)
    h.set_init(w.P)
    bad = w.P[1].copy()
    bad[:, 4] = 0.0
    h.set_init_submodel(3, 1, bad)
    h.iterate(10, 0.0)
    st = h.status()
    assert st["flags"][3] & 2 and not np.any(np.delete(st["flags"], 3) & 2)
    res3 = O.jk_als(w.T, [w.P[0], bad, w.P[2]], p_list=[3], max_iters=10, nthreads=NCPU)
    assert res3.flags[0] & 2
    for a, b in zip(h.factors(3)[0], res3.factors[0]):
        assert rel(a, b) <= 1e-9, rel(a, b)


def test_stress_eight_modes_and_unit_dims():
    # N = 8 (JKCALS_MAX_MODES) with unit-length modes in the middle and a short sampled mode
    from paper_2112_03985_b200 import JKCals
    w = make_workload(((5, 3, 1, 4, 2, 1, 3, 2), 2, 2, 0.01, "syn", 15), seed=8)
    h = JKCals(w.T, w.R, hist_cap=15)
    h.set_init(w.P)
    h.iterate(15, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=15, nthreads=NCPU)
    for p in range(5):
        for a, b in zip(h.factors(p)[0], res.factors[p]):
            assert rel(a, b) <= 1e-10, (p, rel(a, b))


def test_stress_wide_fused_width():
    # a wide fused multi-factor: 268 submodels x R = 20 = 5360 columns (42 M tiles), EEM shape
    from paper_2112_03985_b200 import JKCals
    w = make_workload(((268, 40, 30), 20, 20, 0.02, "eem", 6), seed=2)
    h = JKCals(w.T, w.R, hist_cap=6)
    h.set_init(w.P)
    h.iterate(6, 0.0)
    ps = [0, 133, 267]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=6, nthreads=NCPU)
    for q, p in enumerate(ps):
        for a, b in zip(h.factors(p)[0], res.factors[q]):
            assert rel(a, b) <= 1e-10, (p, rel(a, b))
