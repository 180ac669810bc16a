"""ctypes binding of the ORACLE (test infrastructure, never the product path).

Loads oracle/liborc.so built from jkals_oracle.c (plain C, fp64, pthreads). Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module. It shares no code with paper_2112_03985_b200/.

Arrays crossing this boundary are numpy float64 in column-major (Fortran) order,
matching the oracle's conventions (Eq. 3, first index fastest).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jkals_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

F_CONVERGED, F_PINV, F_NONFINITE, F_BREAKDOWN = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "jkals_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC,
                               "-lpthread", "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        D, I64, I = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        sig = {
            "orc_unfold_index": (None, [I, P, I, P, P, P]),
            "orc_unfold": (None, [I, P, P, I, P]),
            "orc_khatri_rao": (None, [P, I64, P, I64, I, P]),
            "orc_mttkrp_brute": (None, [I, P, P, P, I, I, P]),
            "orc_mttkrp_reference": (None, [I, P, P, P, I, I, P]),
            "orc_gramian": (None, [P, I64, I, P]),
            "orc_hadamard_gramians": (None, [I, P, P, I, I, P]),
            "orc_cholesky_solve": (I, [P, I, P, I64, P]),
            "orc_pinv_solve": (None, [P, I, P, I64, D, P]),
            "orc_norm_sq": (D, [I64, P]),
            "orc_slice_norms_sq": (None, [I, P, P, I, P]),
            "orc_remove_slice": (None, [I, P, P, I, I64, P]),
            "orc_cp_error": (D, [D, P, P, P, I64, I]),
            "orc_explicit_residual": (D, [I, P, P, P, P, I]),
            "orc_cp_als": (I, [I, P, P, I, P, P, I, D, P, P]),
            "orc_jk_als": (I, [I, P, P, I, P, P, I64, I, D, I, P, P, P, P, P]),
            "orc_jk_als_d": (I, [I, P, P, I, P, I64, P, I64, I, D, I, P, P, P, P, P]),
            "orc_remove_slices": (None, [I, P, P, I, I64, I64, P]),
            "orc_align": (I, [I, P, I, P, P, P, P, P, P, P]),
            "orc_jackknife_stats": (I, [I64, I64, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dims(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr_array(mats):
    arr = (ctypes.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
    return arr


def unfold_index(dims, n, idx):
    d = _dims(dims)
    ix = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    row, col = ctypes.c_int64(), ctypes.c_int64()
    lib().orc_unfold_index(len(d), _p(d), n, _p(ix), ctypes.byref(row), ctypes.byref(col))
    return row.value, col.value


def unfold(T, n):
    T = _f64(T)
    d = _dims(T.shape)
    out = np.zeros((d[n], T.size // d[n]), order="F")
    lib().orc_unfold(len(d), _p(d), _p(T), n, _p(out))
    return out


def khatri_rao(A, B):
    A, B = _f64(A), _f64(B)
    assert A.shape[1] == B.shape[1]
    out = np.zeros((A.shape[0] * B.shape[0], A.shape[1]), order="F")
    lib().orc_khatri_rao(_p(A), A.shape[0], _p(B), B.shape[0], A.shape[1], _p(out))
    return out


def mttkrp(T, U, n, path="brute"):
    T = _f64(T)
    U = [_f64(u) for u in U]
    d = _dims(T.shape)
    R = U[0].shape[1]
    out = np.zeros((d[n], R), order="F")
    fn = lib().orc_mttkrp_brute if path == "brute" else lib().orc_mttkrp_reference
    fn(len(d), _p(d), _p(T), _ptr_array(U), R, n, _p(out))
    return out


def gramian(U):
    U = _f64(U)
    G = np.zeros((U.shape[1], U.shape[1]), order="F")
    lib().orc_gramian(_p(U), U.shape[0], U.shape[1], _p(G))
    return G


def hadamard_gramians(U, n):
    U = [_f64(u) for u in U]
    d = _dims([u.shape[0] for u in U])
    R = U[0].shape[1]
    H = np.zeros((R, R), order="F")
    lib().orc_hadamard_gramians(len(d), _p(d), _ptr_array(U), R, n, _p(H))
    return H


def cholesky_solve(H, M):
    H, M = _f64(H), _f64(M)
    U = np.zeros_like(M, order="F")
    rc = lib().orc_cholesky_solve(_p(H), H.shape[0], _p(M), M.shape[0], _p(U))
    return (U if rc == 0 else None)


def pinv_solve(H, M, rcond=1e-12):
    H, M = _f64(H), _f64(M)
    U = np.zeros_like(M, order="F")
    lib().orc_pinv_solve(_p(H), H.shape[0], _p(M), M.shape[0], rcond, _p(U))
    return U


def norm_sq(T):
    T = _f64(T)
    return lib().orc_norm_sq(T.size, _p(T))


def slice_norms_sq(T, mode):
    T = _f64(T)
    d = _dims(T.shape)
    out = np.zeros(d[mode])
    lib().orc_slice_norms_sq(len(d), _p(d), _p(T), mode, _p(out))
    return out


def remove_slice(T, mode, p):
    T = _f64(T)
    d = _dims(T.shape)
    shp = list(T.shape)
    shp[mode] -= 1
    out = np.zeros(shp, order="F")
    lib().orc_remove_slice(len(d), _p(d), _p(T), mode, p, _p(out))
    return out


def remove_slices(T, mode, p0, p1):
    """Delete-d tensor subsample: drop slices p0 <= i_mode < p1."""
    T = _f64(T)
    d = _dims(T.shape)
    shp = list(T.shape)
    shp[mode] -= p1 - p0
    out = np.zeros(shp, order="F")
    lib().orc_remove_slices(len(d), _p(d), _p(T), mode, p0, p1, _p(out))
    return out


def delete_d_groups(I, d):
    """ceil(I/d) contiguous groups of mode-0 indices, the last possibly smaller."""
    return [list(range(g * d, min(g * d + d, I))) for g in range((I + d - 1) // d)]


def cp_error(normT2, H, M, V):
    H, M, V = _f64(H), _f64(M), _f64(V)
    return lib().orc_cp_error(normT2, _p(H), _p(M), _p(V), V.shape[0], V.shape[1])


def explicit_residual(T, U, lam=None):
    T = _f64(T)
    U = [_f64(u) for u in U]
    d = _dims(T.shape)
    lp = None
    if lam is not None:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        lp = _p(lam)
    return lib().orc_explicit_residual(len(d), _p(d), _p(T), _ptr_array(U), lp, U[0].shape[1])


def cp_als(T, U0, max_iters, tol=0.0):
    """Alg. 1 CP-ALS. Returns (U list, lambda, err_hist[:iters], iters, flags)."""
    T = _f64(T)
    U = [np.array(u, dtype=np.float64, order="F", copy=True) for u in U0]
    d = _dims(T.shape)
    R = U[0].shape[1]
    lam = np.zeros(R)
    hist = np.full(max_iters, np.nan)
    iters = ctypes.c_int()
    flags = lib().orc_cp_als(len(d), _p(d), _p(T), R, _ptr_array(U), _p(lam), max_iters, tol,
                             _p(hist), ctypes.byref(iters))
    return U, lam, hist[: iters.value], iters.value, flags


class JKResult:
    """Per-submodel outputs of JK-ALS, indexed by position q in p_list."""

    def __init__(self, dims, R, p_list, U, lam, err, iters, flags, d=1):
        self.dims, self.R, self.p_list, self.d = list(dims), R, list(p_list), d
        self.lam, self.err, self.iters, self.flags = lam, err, iters, flags
        self.factors = []
        for q, g in enumerate(p_list):
            size = min(g * d + d, dims[0]) - g * d
            rows = [dims[0] - size] + list(dims[1:])
            off, fs = 0, []
            for r_ in rows:
                fs.append(U[q, off:off + r_ * R].reshape((r_, R), order="F"))
                off += r_ * R
            self.factors.append(fs)

    def history(self, q):
        return self.err[q, : self.iters[q]]


def jk_als(T, P, p_list=None, max_iters=100, tol=0.0, nthreads=None):
    """Alg. 2 JK-ALS over left-out indices p_list of mode 0 (default: all)."""
    T = _f64(T)
    P = [_f64(u) for u in P]
    d = _dims(T.shape)
    R = P[0].shape[1]
    if p_list is None:
        p_list = range(d[0])
    pl = np.ascontiguousarray(np.asarray(list(p_list), dtype=np.int64))
    npl = len(pl)
    stride = R * (int(d[0]) - 1 + int(d[1:].sum()))
    U = np.zeros((max(npl, 1), stride))
    lam = np.zeros((max(npl, 1), R))
    err = np.zeros((max(npl, 1), max_iters))
    iters = np.zeros(max(npl, 1), dtype=np.int32)
    flags = np.zeros(max(npl, 1), dtype=np.int32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib().orc_jk_als(len(d), _p(d), _p(T), R, _ptr_array(P), _p(pl), npl, max_iters, tol,
                          nthreads, _p(U), _p(lam), _p(err), _p(iters), _p(flags))
    if rc != 0:
        raise ValueError("orc_jk_als rejected its arguments")
    return JKResult(d.tolist(), R, pl.tolist(), U, lam, err, iters, flags)


def jk_als_d(T, P, d, g_list=None, max_iters=100, tol=0.0, nthreads=None):
    """Delete-d JK-ALS: group g removes mode-0 rows [g*d, min(g*d+d, I_0))."""
    T = _f64(T)
    P = [_f64(u) for u in P]
    dims = _dims(T.shape)
    R = P[0].shape[1]
    if d < 1:
        raise ValueError("delete-d needs d >= 1")
    ngroups = (int(dims[0]) + d - 1) // d
    if g_list is None:
        g_list = range(ngroups)
    gl = np.ascontiguousarray(np.asarray(list(g_list), dtype=np.int64))
    ng = len(gl)
    stride = R * (int(dims[0]) - 1 + int(dims[1:].sum()))
    U = np.zeros((max(ng, 1), stride))
    lam = np.zeros((max(ng, 1), R))
    err = np.zeros((max(ng, 1), max_iters))
    iters = np.zeros(max(ng, 1), dtype=np.int32)
    flags = np.zeros(max(ng, 1), dtype=np.int32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib().orc_jk_als_d(len(dims), _p(dims), _p(T), R, _ptr_array(P), d, _p(gl), ng, max_iters,
                            tol, nthreads, _p(U), _p(lam), _p(err), _p(iters), _p(flags))
    if rc != 0:
        raise ValueError("orc_jk_als_d rejected its arguments")
    return JKResult(dims.tolist(), R, gl.tolist(), U, lam, err, iters, flags, d=d)


def jackknife_stats(X):
    """X: (g, ...) stack of per-submodel matrices -> (mean, std) with the (g-1)/g factor."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    g = X.shape[0]
    ln = X[0].size
    mean = np.zeros(ln)
    std = np.zeros(ln)
    rc = lib().orc_jackknife_stats(g, ln, _p(X), _p(mean), _p(std))
    if rc != 0:
        raise ValueError("jackknife stats need g >= 2")
    return mean.reshape(X.shape[1:]), std.reshape(X.shape[1:])


def align(Uh, lam, P):
    """Alg. 2 alg:jk:perm_scale with DESIGN.md reading A12: returns
    (aligned factors, perm (R,), sign (N, R), congruence (R,))."""
    Uh = [_f64(u) for u in Uh]
    P = [_f64(p) for p in P]
    N, R = len(Uh), Uh[0].shape[1]
    rows = np.ascontiguousarray([u.shape[0] for u in Uh], dtype=np.int64)
    out = [np.zeros(u.shape, order="F") for u in Uh]
    perm = np.zeros(R, dtype=np.int32)
    sign = np.zeros((N, R), dtype=np.int32)
    cong = np.zeros(R)
    lp = None
    if lam is not None:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        lp = _p(lam)
    rc = lib().orc_align(N, _p(rows), R, _ptr_array(Uh), lp, _ptr_array(P), _ptr_array(out), _p(perm),
                         _p(sign), _p(cong))
    if rc != 0:
        raise ValueError("orc_align rejected its arguments")
    return out, perm, sign, cong


def mode0_full(U0, group, I0):
    """A submodel's mode-0 factor ((I0 - |group|) x R) re-indexed to the I0 global rows, the
    group's rows NaN (absent)."""
    R = U0.shape[1]
    out = np.full((I0, R), np.nan)
    keep = [i for i in range(I0) if i not in set(group)]
    out[keep] = U0
    return out


def present_stats(X):
    """Jackknife mean and SE per element over the submodels in which the element is present
    (X: (g, ...) with NaN = absent; reading A20 for the sampled mode):
    g_e = present count, std = sqrt(((g_e - 1)/g_e) sum (x - mean)^2); elements with g_e < 2
    get std = 0 (and mean = the value, or 0 if absent everywhere)."""
    X = np.asarray(X, dtype=np.float64)
    g = X.shape[0]
    flat = X.reshape(g, -1)
    mean = np.zeros(flat.shape[1])
    std = np.zeros(flat.shape[1])
    cnt = np.zeros(flat.shape[1])
    for e in range(flat.shape[1]):
        vals = [flat[q, e] for q in range(g) if not np.isnan(flat[q, e])]
        cnt[e] = len(vals)
        if not vals:
            continue
        mu = sum(vals) / len(vals)
        mean[e] = mu
        if len(vals) >= 2:
            ss = sum((v - mu) * (v - mu) for v in vals)
            std[e] = np.sqrt(((len(vals) - 1) / len(vals)) * ss)
    shp = X.shape[1:]
    return mean.reshape(shp), std.reshape(shp), cnt.reshape(shp)
