"""Pins for the oracle (CPU only, `-m "not gpu"`).

The oracle (oracle/jkals_oracle.c) must be pinned to something other than itself:
SPEC/paper examples, closed forms, invariants, library routines (numpy) for special
cases, and brute force on tiny inputs. Each test names the passage it checks.
"""
import numpy as np
import pytest

from oracle import oracle as O
from synth import make_workload
from synth.workloads import compose, make_tensor


def rng(seed=0):
    return np.random.default_rng(seed)


def np_unfold(T, n):
    """Kolda unfolding via numpy (library routine; independent of the oracle)."""
    return np.reshape(np.moveaxis(T, n, 0), (T.shape[n], -1), order="F")


def np_krp(mats):
    """Descending-order KRP U_{N-1} (.) ... (.) U_0 via numpy kron per column."""
    R = mats[0].shape[1]
    cols = []
    for r in range(R):
        c = np.ones(1)
        for m in mats:  # ascending m; kron(m, c) puts the earlier modes fastest
            c = np.kron(m[:, r], c)
        cols.append(c)
    return np.stack(cols, axis=1)


# ---------------------------------------------------------------- unfolding (Eq. 3)
def test_unfold_index_spec_examples():
    # SPEC.md:46-48 (1-based): dims (2,3,2), n=1, (2,3,1) -> (2,3); n=2, (2,3,2) -> (3,4)
    assert O.unfold_index((2, 3, 2), 0, (1, 2, 0)) == (1, 2)
    assert O.unfold_index((2, 3, 2), 0, (0, 0, 0)) == (0, 0)
    assert O.unfold_index((2, 3, 2), 1, (1, 2, 1)) == (2, 3)


@pytest.mark.parametrize("dims", [(2, 3, 2), (3, 4, 5), (2, 3, 4, 2)])
def test_unfold_matches_numpy_moveaxis(dims):
    # PAPER.md:196 + Eq. 3 vs numpy's Kolda unfolding
    T = np.asfortranarray(rng(1).standard_normal(dims))
    for n in range(len(dims)):
        assert np.array_equal(O.unfold(T, n), np_unfold(T, n))


# ---------------------------------------------------------------- Khatri-Rao
def test_khatri_rao_spec_examples():
    # SPEC.md:64-66
    assert np.array_equal(O.khatri_rao([[1.0], [2.0]], [[3.0], [4.0]]).ravel(), [3, 4, 6, 8])
    A = rng(2).standard_normal((4, 3))
    assert np.array_equal(O.khatri_rao(A, np.ones((1, 3))), A)


def test_khatri_rao_matches_numpy_kron():
    A, B = rng(3).standard_normal((3, 2)), rng(4).standard_normal((4, 2))
    ref = np.stack([np.kron(A[:, r], B[:, r]) for r in range(2)], axis=1)
    assert np.array_equal(O.khatri_rao(A, B), ref)


# ---------------------------------------------------------------- MTTKRP
@pytest.mark.parametrize("dims", [(4, 3, 2), (3, 4, 4, 2), (5, 4, 3)])
def test_mttkrp_brute_vs_reference_vs_numpy(dims):
    # Alg. 1 alg:als:mttkrp, Eq. 1: brute force over every
    # element == explicit unfolding x explicit KRP == numpy (unfold @ kron-KRP).
    g = rng(5)
    T = np.asfortranarray(g.standard_normal(dims))
    R = 3
    U = [g.standard_normal((I, R)) for I in dims]
    for n in range(len(dims)):
        mb = O.mttkrp(T, U, n, "brute")
        mr = O.mttkrp(T, U, n, "reference")
        mn = np_unfold(T, n) @ np_krp([U[m] for m in range(len(dims)) if m != n])
        assert np.allclose(mb, mr, rtol=1e-13, atol=1e-13)
        assert np.allclose(mb, mn, rtol=1e-13, atol=1e-13)


def test_mttkrp_zero_factors_and_rank1():
    # zero factors -> 0; T = a o b o c, unit-norm b, c -> M_1 = a
    g = rng(6)
    a, b, c = g.standard_normal(5), g.standard_normal(4), g.standard_normal(3)
    b /= np.linalg.norm(b)
    c /= np.linalg.norm(c)
    T = np.asfortranarray(np.einsum("i,j,k->ijk", a, b, c))
    U = [np.zeros((5, 1)), b[:, None], c[:, None]]
    assert np.allclose(O.mttkrp(T, U, 0)[:, 0], a, atol=1e-14)
    Z = [np.zeros((5, 2)), np.zeros((4, 2)), np.zeros((3, 2))]
    assert np.all(O.mttkrp(T, Z, 1) == 0)


def test_case_I_and_II_zero_row_invariant():
    # §4.1: with row p of U_0 zeroed, the full-tensor MTTKRP equals the
    # sliced-tensor MTTKRP for n != 0 (Case II) -- bitwise, as the same terms are summed
    # in the same order plus exact zeros -- and for n = 0 all rows != p agree (Case I).
    g = rng(7)
    dims, R, p = (6, 5, 4), 3, 2
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, R)) for I in dims]
    Tp = O.remove_slice(T, 0, p)
    Up = [np.delete(U[0], p, axis=0)] + U[1:]
    Uz = [U[0].copy()] + U[1:]
    Uz[0][p] = 0.0
    for n in (1, 2):
        assert np.array_equal(O.mttkrp(T, Uz, n), O.mttkrp(Tp, Up, n))
    m_full = O.mttkrp(T, U, 0)
    m_sub = O.mttkrp(Tp, Up, 0)
    assert np.allclose(np.delete(m_full, p, axis=0), m_sub, rtol=1e-14, atol=1e-14)


# ---------------------------------------------------------------- Gramians, solves
def test_hadamard_gramians_closed_forms():
    # orthonormal -> I ; all-ones -> prod_{i != n} I_i
    g = rng(8)
    Q = [np.linalg.qr(g.standard_normal((I, 3)))[0] for I in (5, 6, 7)]
    assert np.allclose(O.hadamard_gramians(Q, 0), np.eye(3), atol=1e-14)
    ones = [np.ones((I, 2)) for I in (3, 4, 5)]
    assert np.array_equal(O.hadamard_gramians(ones, 1), np.full((2, 2), 15.0))
    A = g.standard_normal((9, 4))
    assert np.allclose(O.gramian(A), A.T @ A, rtol=1e-14)


def test_solves():
    g = rng(9)
    M = g.standard_normal((7, 3))
    assert np.allclose(O.cholesky_solve(np.eye(3), M), M)
    # H = diag(2,0), M = [2 4; 6 8] -> [1 0; 3 0]
    assert np.allclose(O.pinv_solve(np.diag([2.0, 0.0]), [[2.0, 4.0], [6.0, 8.0]]),
                       [[1.0, 0.0], [3.0, 0.0]], atol=1e-15)
    A = g.standard_normal((10, 3))
    H = A.T @ A
    U = O.cholesky_solve(H, M)
    assert np.allclose(U @ H, M, rtol=1e-10, atol=1e-12)          # residual identity
    assert np.allclose(U, M @ np.linalg.inv(H), rtol=1e-12)       # library routine
    assert np.allclose(O.pinv_solve(H, M), U, rtol=1e-10)          # Cholesky == pinv
    assert np.allclose(O.pinv_solve(H, M), M @ np.linalg.pinv(H), rtol=1e-10)
    assert O.cholesky_solve(np.diag([1.0, -1.0, 2.0]), M) is None  # not SPD -> fallback


def test_slice_norms_and_remove_slice():
    # SPEC.md:110-121
    T = np.ones((2, 2, 2), order="F")
    assert O.norm_sq(T) == 8.0
    assert np.array_equal(O.slice_norms_sq(T, 0), [4.0, 4.0])
    g = rng(10)
    T = np.asfortranarray(g.standard_normal((5, 3, 2)))
    assert np.isclose(O.slice_norms_sq(T, 0).sum(), O.norm_sq(T), rtol=1e-13)
    assert np.array_equal(O.remove_slice(T, 0, 1), np.delete(T, 1, axis=0))
    assert np.array_equal(O.remove_slice(T, 1, 2), np.delete(T, 2, axis=1))


# ---------------------------------------------------------------- error formula
def test_error_formula_sign_and_explicit_residual():
    # Alg. 1 alg:als:error with "+": at the LS update of the
    # last mode, e equals the explicit residual ||T - [[U]]||^2; the printed "-" does not.
    g = rng(11)
    dims, R = (6, 5, 4), 3
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, R)) for I in dims]
    n = 2
    M = O.mttkrp(T, U, n)
    H = O.hadamard_gramians(U, n)
    V = M @ np.linalg.inv(H)
    e = O.cp_error(O.norm_sq(T), H, M, V)
    Ue = U[:2] + [V]
    res = O.explicit_residual(T, Ue)
    dense = np.einsum("ir,jr,kr->ijk", *Ue)
    assert np.isclose(res, np.sum((T - dense) ** 2), rtol=1e-12)
    assert np.isclose(e, res, rtol=1e-10)
    wrong = O.norm_sq(T) - np.sum(H * (V.T @ V)) - 2 * np.sum(V * M)
    assert not np.isclose(wrong, res, rtol=1e-3)
    # zero model -> ||T||^2 ; exact model -> 0
    Z = np.zeros_like(V)
    assert O.cp_error(O.norm_sq(T), H, M, Z) == O.norm_sq(T)


# ---------------------------------------------------------------- CP-ALS
def test_cp_als_monotone_and_explicit_error():
    # SPEC.md:209 monotone non-increasing error; error history equals explicit residual
    w = make_workload(((9, 8, 7), 3, 4, 0.1, "syn", 30), seed=3)
    U, lam, hist, iters, flags = O.cp_als(w.T, w.P, 30)
    assert iters == 30 and flags == 0
    n2 = O.norm_sq(w.T)
    assert np.all(np.diff(hist) <= 1e-12 * n2)
    assert np.isclose(hist[-1], O.explicit_residual(w.T, U, lam), rtol=1e-8)


def test_cp_als_fixed_point_and_exact_recovery():
    # exact noiseless factors are a fixed point; noiseless planted
    # tensor is recovered (error < 1e-6 ||T||^2 within 200 sweeps).
    T, A = make_tensor((10, 12, 14), 2, 0.0, "syn", seed=4)
    n2 = O.norm_sq(T)
    U, lam, hist, _, _ = O.cp_als(T, A, 5)
    assert abs(hist[-1]) < 1e-12 * n2  # fast formula cancels to rounding level
    rec = compose([U[0] * lam] + U[1:])
    assert np.allclose(rec, T, rtol=1e-10, atol=1e-12)
    g = rng(12)
    P = [a + 0.2 * g.standard_normal(a.shape) for a in A]
    U, lam, hist, _, _ = O.cp_als(T, P, 200)
    assert hist[-1] < 1e-6 * n2


def test_cp_als_rank1_closed_form():
    # T = a o b o c, R = 1: one sweep gives columns proportional to a, b, c
    g = rng(13)
    a, b, c = g.uniform(0.5, 1, 6), g.uniform(0.5, 1, 5), g.uniform(0.5, 1, 4)
    T = np.asfortranarray(np.einsum("i,j,k->ijk", a, b, c))
    P = [g.uniform(0.1, 1, (6, 1)), g.uniform(0.1, 1, (5, 1)), g.uniform(0.1, 1, (4, 1))]
    U, lam, hist, _, _ = O.cp_als(T, P, 1)
    for u, v in zip(U, (a, b, c)):
        assert np.allclose(u[:, 0], v / np.linalg.norm(v), rtol=1e-12)
    assert np.isclose(lam[0], np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(c))


def test_cp_als_initial_mode0_irrelevant():
    # mode 0 is updated first from U_1..U_{N-1}, so U_0's initial value
    # never enters the trajectory.
    w = make_workload("tiny")
    P2 = [np.full_like(w.P[0], 7.0)] + w.P[1:]
    h1 = O.cp_als(w.T, w.P, 10)[2]
    h2 = O.cp_als(w.T, P2, 10)[2]
    assert np.array_equal(h1, h2)


def test_cp_als_tolerance_rule():
    # stop when |fit - fit_prev| < tol, tested from sweep 2
    w = make_workload("tiny")
    _, _, hist, iters, flags = O.cp_als(w.T, w.P, 1000, tol=1e-6)
    assert flags & O.F_CONVERGED and 2 <= iters < 1000 and len(hist) == iters
    _, _, _, iters, _ = O.cp_als(w.T, w.P, 1000, tol=1e300)
    assert iters == 2


# ---------------------------------------------------------------- JK-ALS
def test_jk_als_matches_manual_slicing():
    # Alg. 2: submodel p is cp_als on T_-p from P with row p dropped
    w = make_workload("tiny")
    res = O.jk_als(w.T, w.P, p_list=[0, 4, 9], max_iters=20, nthreads=3)
    for q, p in enumerate([0, 4, 9]):
        Tp = O.remove_slice(w.T, 0, p)
        Pp = [np.delete(w.P[0], p, axis=0)] + w.P[1:]
        U, lam, hist, _, _ = O.cp_als(Tp, Pp, 20)
        for a, b in zip(res.factors[q], U):
            assert np.array_equal(a, b)
        assert np.array_equal(res.history(q), hist)
        assert np.array_equal(res.lam[q], lam)


def test_jk_threads_deterministic():
    # thread count does not change per-submodel results
    w = make_workload("tiny")
    r1 = O.jk_als(w.T, w.P, max_iters=10, nthreads=1)
    r4 = O.jk_als(w.T, w.P, max_iters=10, nthreads=4)
    assert np.array_equal(r1.err, r4.err)


def test_jackknife_stats():
    # identical -> 0 ; two-point v +/- d -> d ; numpy: sqrt(g-1)*std
    X = np.ones((5, 3, 2))
    m, s = O.jackknife_stats(X)
    assert np.all(s == 0) and np.all(m == 1)
    X = np.array([[1.0 + 0.25], [1.0 - 0.25]])
    assert np.isclose(O.jackknife_stats(X)[1][0], 0.25)
    X = rng(14).standard_normal((7, 4, 3))
    assert np.allclose(O.jackknife_stats(X)[1], np.sqrt(6) * X.std(axis=0), rtol=1e-13)


def _numpy_jk_cals(T, P, sweeps):
    """Test-only JK-CALS (Alg. 3) in numpy on the FULL tensor with zero rows, used to
    make the §4.1 theorem executable against the oracle's JK-ALS."""
    dims = T.shape
    N, I0, R = len(dims), dims[0], P[0].shape[1]
    U = [[p.copy() for p in P] for _ in range(I0)]
    for p in range(I0):
        U[p][0][p] = 0.0
    errs = np.zeros((I0, sweeps))
    for it in range(sweeps):
        for n in range(N):
            Tn = np_unfold(T, n)
            for p in range(I0):
                K = np_krp([U[p][m] for m in range(N) if m != n])
                M = Tn @ K
                H = np.ones((R, R))
                for m in range(N):
                    if m != n:
                        H *= U[p][m].T @ U[p][m]
                V = M @ np.linalg.inv(H)
                if n == 0:
                    V[p] = 0.0
                lam = np.linalg.norm(V, axis=0)
                U[p][n] = V / lam
                if n == N - 1:
                    n2p = np.sum(T * T) - np.sum(T[p] ** 2)
                    errs[p, it] = n2p + np.sum(H * (V.T @ V)) - 2 * np.sum(V * M)
    return U, errs


def test_jk_cals_equals_jk_als_theorem():
    # §4.1 made executable: JK-CALS on the full tensor with zero rows
    # reaches the JK-ALS submodels (tolerance 1e-10 here).
    w = make_workload(((7, 6, 5), 2, 2, 0.05, "syn", 15), seed=5)
    res = O.jk_als(w.T, w.P, max_iters=15)
    U, errs = _numpy_jk_cals(w.T, w.P, 15)
    for p in range(7):
        a = res.factors[p]
        assert np.allclose(np.delete(U[p][0], p, axis=0), a[0], rtol=1e-10, atol=1e-12)
        assert np.all(U[p][0][p] == 0.0)
        for n in (1, 2):
            assert np.allclose(U[p][n], a[n], rtol=1e-10, atol=1e-12)
        assert np.allclose(errs[p], res.history(p), rtol=1e-9)


# ---------------------------------------------------------------- delete-d jackknife (§4.2)
def test_delete_d_groups_partition():
    # ceil(I/d) contiguous disjoint groups covering 0..I-1
    for I, d in [(10, 1), (10, 3), (7, 2), (50, 5), (9, 4)]:
        G = O.delete_d_groups(I, d)
        assert len(G) == -(-I // d)
        assert sum(G, []) == list(range(I))
        assert all(len(g) == d for g in G[:-1]) and 1 <= len(G[-1]) <= d


def test_remove_slices_matches_numpy_delete():
    # PAPER.md:416-417 (delete-d subsample) against numpy.delete (library routine)
    T = rng(21).standard_normal((9, 4, 3))
    T = np.asfortranarray(T)
    for p0, p1 in [(0, 2), (3, 6), (8, 9)]:
        out = O.remove_slices(T, 0, p0, p1)
        assert np.array_equal(out, np.delete(T, range(p0, p1), axis=0))
    assert np.array_equal(O.remove_slices(T, 0, 4, 5), O.remove_slice(T, 0, 4))


def test_jk_als_d1_is_leave_one_out():
    # d = 1 is leave-one-out: identical submodels, bit for bit
    w = make_workload("tiny")
    a = O.jk_als(w.T, w.P, max_iters=12, nthreads=2)
    b = O.jk_als_d(w.T, w.P, 1, max_iters=12, nthreads=2)
    assert np.array_equal(a.err, b.err) and np.array_equal(a.lam, b.lam)
    for fa, fb in zip(a.factors, b.factors):
        for x, y in zip(fa, fb):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("d", [2, 3, 5])
def test_jk_als_d_matches_manual_group_removal(d):
    # Alg. 2 with a group of d rows removed: each group's
    # submodel is cp_als on numpy-deleted T and P_0 (independent of orc_remove_slices)
    w = make_workload("tiny")   # I_0 = 10: d = 3 leaves a ragged last group of 1
    res = O.jk_als_d(w.T, w.P, d, max_iters=15, nthreads=3)
    G = O.delete_d_groups(10, d)
    assert len(res.factors) == len(G)
    for q, g in enumerate(G):
        Tp = np.asfortranarray(np.delete(w.T, g, axis=0))
        Pp = [np.delete(w.P[0], g, axis=0)] + w.P[1:]
        U, lam, hist, _, _ = O.cp_als(Tp, Pp, 15)
        assert res.factors[q][0].shape == (10 - len(g), w.R)
        for a, b in zip(res.factors[q], U):
            assert np.array_equal(a, b)
        assert np.array_equal(res.history(q), hist)


def test_jk_als_d_rejects_bad_d():
    # d <= I/2 and group indices < ceil(I/d)
    w = make_workload("tiny")
    for d in (0, 6):
        with pytest.raises(ValueError):
            O.jk_als_d(w.T, w.P, d, max_iters=2)
    with pytest.raises(ValueError):
        O.jk_als_d(w.T, w.P, 3, g_list=[4], max_iters=2)


def _numpy_jk_cals_d(T, P, d, sweeps):
    """Test-only delete-d JK-CALS: pad and re-zero d rows per group."""
    dims = T.shape
    N, I0, R = len(dims), dims[0], P[0].shape[1]
    G = [list(range(g * d, min(g * d + d, I0))) for g in range(-(-I0 // d))]
    U = [[p.copy() for p in P] for _ in G]
    for q, g in enumerate(G):
        U[q][0][g] = 0.0
    errs = np.zeros((len(G), sweeps))
    for it in range(sweeps):
        for n in range(N):
            Tn = np_unfold(T, n)
            for q, g in enumerate(G):
                M = Tn @ np_krp([U[q][m] for m in range(N) if m != n])
                H = np.ones((R, R))
                for m in range(N):
                    if m != n:
                        H *= U[q][m].T @ U[q][m]
                V = M @ np.linalg.inv(H)
                if n == 0:
                    V[g] = 0.0
                U[q][n] = V / np.linalg.norm(V, axis=0)
                if n == N - 1:
                    n2p = np.sum(T * T) - np.sum(T[g] ** 2)
                    errs[q, it] = n2p + np.sum(H * (V.T @ V)) - 2 * np.sum(V * M)
    return G, U, errs


@pytest.mark.parametrize("d", [2, 3])
def test_delete_d_jk_cals_equals_jk_als(d):
    # §4.2 "pad and periodically zero out d rows" reaches the delete-d
    # JK-ALS submodels (the §4.1 theorem with E_p deleting d rows); I_0 = 7 gives a ragged group
    w = make_workload(((7, 6, 5), 2, 2, 0.05, "syn", 12), seed=9)
    res = O.jk_als_d(w.T, w.P, d, max_iters=12)
    G, U, errs = _numpy_jk_cals_d(w.T, w.P, d, 12)
    for q, g in enumerate(G):
        a = res.factors[q]
        assert np.all(U[q][0][g] == 0.0)
        assert np.allclose(np.delete(U[q][0], g, axis=0), a[0], rtol=1e-10, atol=1e-12)
        for n in (1, 2):
            assert np.allclose(U[q][n], a[n], rtol=1e-10, atol=1e-12)
        assert np.allclose(errs[q], res.history(q), rtol=1e-9)


# ---------------------------------------------------------------- alignment (Alg. 2 line 6)
def _recon(U, lam=None):
    return compose([u * (lam if (lam is not None and k == 0) else 1.0) for k, u in enumerate(U)])


def _unit(U):
    return [u / np.linalg.norm(u, axis=0) for u in U]


def test_align_recovers_column_permutation():
    # SPEC.md:361 self-alignment: P_hat = P with columns permuted -> permutation recovered exactly
    g = rng(31)
    P = [g.uniform(0, 1, (I, 4)) for I in (7, 6, 5)]
    pi = np.array([2, 0, 3, 1])              # P_hat column r = P column pi[r]
    Uh = _unit([p[:, pi] for p in P])
    lam = np.array([1.5, 2.0, 0.5, 3.0])
    out, perm, sign, cong = O.align(Uh, lam, P)
    assert np.array_equal(perm, pi) and np.all(sign == 1)
    assert np.allclose(cong, 1.0, rtol=0, atol=1e-14)
    Pu = _unit(P)
    for n in (1, 2):
        assert np.allclose(out[n], Pu[n], rtol=0, atol=1e-15)
    # mode 0 absorbs lambda: column pi[r] of out_0 = lam_r * Uh_0(:, r)
    for r in range(4):
        assert np.allclose(out[0][:, pi[r]], lam[r] * Uh[0][:, r], rtol=1e-15)


def test_align_sign_flips_restored_model_unchanged():
    # one column negated in two non-sampled modes -> flips undone, tensor unchanged
    g = rng(32)
    P = _unit([g.uniform(0, 1, (I, 3)) for I in (6, 5, 4, 3)])
    Uh = [p.copy() for p in P]
    Uh[1][:, 2] *= -1
    Uh[3][:, 2] *= -1
    out, perm, sign, cong = O.align(Uh, None, P)
    assert np.array_equal(perm, [0, 1, 2])
    assert sign[1, 2] == -1 and sign[3, 2] == -1 and sign[0, 2] == 1 and sign[2, 2] == 1
    for n in range(4):
        assert np.allclose(out[n], P[n], rtol=0, atol=1e-15)
    # an odd number of flips is compensated in mode 0
    Uh = [p.copy() for p in P]
    Uh[2][:, 0] *= -1
    out, _, sign, _ = O.align(Uh, None, P)
    assert sign[0, 0] == -1 and sign[2, 0] == -1
    assert np.allclose(out[0][:, 0], -Uh[0][:, 0]) and np.allclose(out[2][:, 0], P[2][:, 0])


def test_align_reconstruction_invariant_and_congruent():
    # alignment never changes the model's tensor (<= 1e-12 relative); afterwards
    # every non-sampled column has unit norm and non-negative cosine with its reference column
    g = rng(33)
    for R in (1, 2, 5, 7):
        P = [g.uniform(0, 1, (I, R)) for I in (8, 7, 6)]
        pi = g.permutation(R)
        Uh = [p[:, pi] + 0.2 * g.standard_normal((p.shape[0], R)) for p in P]
        Uh[1][:, 0] *= -1
        lam = g.uniform(0.5, 2, R)
        out, perm, sign, cong = O.align(Uh, lam, P)
        T0 = _recon(Uh, lam)
        assert np.linalg.norm(_recon(out) - T0) <= 1e-12 * np.linalg.norm(T0)
        for n in (1, 2):
            assert np.allclose(np.linalg.norm(out[n], axis=0), 1.0, atol=1e-14)
            assert np.all(np.sum(out[n] * P[n], axis=0) >= 0)
        assert sorted(perm.tolist()) == list(range(R))


def test_align_assignment_matches_scipy():
    # the exhaustive lexicographic search finds the same optimum as scipy's linear_sum_assignment
    # (a library routine) on the congruence matrix
    from scipy.optimize import linear_sum_assignment
    g = rng(34)
    for trial in range(10):
        R = int(g.integers(2, 9))
        P = [g.standard_normal((I, R)) for I in (5, 9, 8)]
        Uh = [g.standard_normal((I, R)) for I in (5, 9, 8)]
        _, perm, _, cong = O.align(Uh, None, P)
        C = np.ones((R, R))
        for n in (1, 2):
            a = Uh[n] / np.linalg.norm(Uh[n], axis=0)
            b = P[n] / np.linalg.norm(P[n], axis=0)
            C *= np.abs(a.T @ b)
        r_, c_ = linear_sum_assignment(C, maximize=True)
        assert np.isclose(C[r_, c_].sum(), sum(C[r, perm[r]] for r in range(R)), rtol=1e-13)
        assert np.array_equal(perm, c_[np.argsort(r_)])


def test_present_stats():
    # sampled-mode stats over the submodels in which a row is present (A20):
    # a row missing from one of g submodels has g-1 contributions; two-point case -> delta
    X = np.array([[[1.0], [np.nan]], [[3.0], [5.0]], [[np.nan], [7.0]]])
    m, s, c = O.present_stats(X)
    assert np.array_equal(c[:, 0], [2, 2])
    assert np.allclose(m[:, 0], [2.0, 6.0]) and np.allclose(s[:, 0], [1.0, 1.0])
    Y = rng(35).standard_normal((6, 4, 2))
    m2, s2, c2 = O.present_stats(Y)
    mj, sj = O.jackknife_stats(Y)
    assert np.allclose(m2, mj, rtol=1e-14) and np.allclose(s2, sj, rtol=1e-13) and np.all(c2 == 6)


def test_mode0_full_reindexing():
    # a submodel's mode-0 factor without its group's rows, put back on the I_0 global rows
    U0 = np.arange(14.0).reshape(7, 2)
    F = O.mode0_full(U0, [3, 4, 5], 10)
    assert np.all(np.isnan(F[3:6])) and np.array_equal(F[:3], U0[:3]) and np.array_equal(F[6:], U0[3:])
