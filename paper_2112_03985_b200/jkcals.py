"""Thin Python binding of the JK-CALS C ABI (include/jkcals.h).

Argument marshalling only: every step of the hot path runs in libjkcals.so (CUDA,
sm_100a). PyTorch provides device memory (the workspace), the CUDA stream and, in
dist.py, process groups. There is no CPU fallback: if the library or a CUDA device
is missing, every entry point raises.

Names follow the paper (arXiv 2112.03985): T the target tensor, P the overall model
(warm start), submodel p leaves out slice p of the sampled mode 0.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

FP64, FP32, FP64_I8 = 0, 1, 2  # FP64_I8: experimental INT8-sliced MTTKRP
F_CONVERGED, F_PINV_FALLBACK, F_NONFINITE, F_BREAKDOWN = 1, 2, 4, 8
DEFAULT_TOL, DEFAULT_MAX_ITERS = 1e-6, 1000  # PAPER.md:596, 608 (§5.2 protocol)

_STATUS = {0: "OK", -1: "E_ARG", -2: "E_SHAPE", -3: "E_STATE", -4: "E_OOM", -5: "E_CUDA", -6: "E_NONFINITE"}


class JKCalsError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"jkcals {_STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libjkcals.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        path = os.environ.get("JKCALS_LIB")  # dev A/B timing of another build of the same ABI
        if not path:
            path = _build.LIB
            if _build.stale():
                path = _build.build()
        L = ctypes.CDLL(path)
        P, I, I64, D, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
        sigs = {
            "jkcals_workspace_bytes": (SZ, [I, P, I, I64, I, I, I]),
            "jkcals_create": (I, [P, I, P, I, I64, I64, P, I, I, I, P, P, SZ, I]),
            "jkcals_create_d": (I, [P, I, P, I, I64, I64, I64, P, I, I, I, P, P, SZ, I]),
            "jkcals_pool_workspace_bytes": (SZ, [I, P, I, P, I64, I64, I64, I, I, I]),
            "jkcals_create_pool": (I, [P, I, P, I, P, I64, I64, I64, P, I, I, I, P, P, SZ, I]),
            "jkcals_get_model_stats": (I, [P, I, I, P, P]),
            "jkcals_get_model_moments": (I, [P, I, I, P, P, P]),
            "jkcals_align": (I, [P]),
            "jkcals_config_workspace_bytes": (SZ, [P]),
            "jkcals_create_config": (I, [P, P, P, I, P, P, SZ]),
            "jkcals_num_slots": (I, [P]),
            "jkcals_get_ids": (I, [P, P]),
            "jkcals_state_bytes": (SZ, [P, I64]),
            "jkcals_export_submodel": (I, [P, I64, P, SZ]),
            "jkcals_import_submodel": (I, [P, P, SZ]),
            "jkcals_get_alignment": (I, [P, I64, P, P, P]),
            "jkcals_get_aligned_factors": (I, [P, I64, I, P]),
            "jkcals_get_aligned_moments": (I, [P, I, I, P, P, P]),
            "jkcals_get_aligned_stats": (I, [P, I, I, P, P]),
            "jkcals_set_init": (I, [P, P]),
            "jkcals_set_init_submodel": (I, [P, I64, I, P]),
            "jkcals_set_init_all": (I, [P, I, P]),
            "jkcals_iterate": (I, [P, I, D, P]),
            "jkcals_get_factors": (I, [P, I64, I, P, P]),
            "jkcals_get_block": (I, [P, I64, I, P]),
            "jkcals_get_all_factors": (I, [P, I, P, P]),
            "jkcals_get_status": (I, [P, P, P, P, P]),
            "jkcals_get_history": (I, [P, I64, P, I, P]),
            "jkcals_get_jackknife_stats": (I, [P, I, P, P]),
            "jkcals_get_local_moments": (I, [P, I, P, P, P]),
            "jkcals_set_instrument": (I, [P, I]),
            "jkcals_get_kernel_times": (I, [P, P, P, P]),
            "jkcals_sweep_flops": (D, [P]),
            "jkcals_launches_per_sweep": (I, [P]),
            "jkcals_last_error": (ctypes.c_char_p, [P]),
            "jkcals_destroy": (None, [P]),
            "jkcals_mttkrp_scratch_bytes": (SZ, [I, P, I, I64, I]),
            "jkcals_mttkrp": (I, [I, P, I, P, P, I64, I64, P, I64, P, SZ, P]),
            "jkcals_mttkrp_i8_scratch_bytes": (SZ, [I, P, I, I64, I]),
            "jkcals_mttkrp_i8": (I, [I, P, I, P, P, I64, I64, P, I64, P, SZ, P]),
            "jkcals_krp": (I, [I, P, I, P, I64, I64, P, I64, P]),
            "jkcals_merge_moments": (I, [I, I64, P, P, P, P, P, P]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


EXPORTED = [
    "jkcals_workspace_bytes", "jkcals_create", "jkcals_create_d", "jkcals_pool_workspace_bytes",
    "jkcals_create_pool", "jkcals_get_model_stats", "jkcals_get_model_moments", "jkcals_align",
    "jkcals_set_init_all", "jkcals_config_workspace_bytes", "jkcals_mttkrp_i8_scratch_bytes", "jkcals_mttkrp_i8", "jkcals_create_config", "jkcals_num_slots", "jkcals_get_ids",
    "jkcals_state_bytes", "jkcals_export_submodel", "jkcals_import_submodel",
    "jkcals_get_alignment", "jkcals_get_aligned_factors", "jkcals_get_aligned_moments", "jkcals_get_aligned_stats",
    "jkcals_set_init", "jkcals_set_init_submodel", "jkcals_iterate",
    "jkcals_get_factors", "jkcals_get_all_factors", "jkcals_get_block", "jkcals_get_status", "jkcals_get_history", "jkcals_get_jackknife_stats",
    "jkcals_get_local_moments", "jkcals_set_instrument", "jkcals_get_kernel_times", "jkcals_sweep_flops",
    "jkcals_launches_per_sweep", "jkcals_last_error", "jkcals_destroy", "jkcals_mttkrp_scratch_bytes",
    "jkcals_mttkrp", "jkcals_krp", "jkcals_merge_moments",
]


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise JKCalsError(-5, "no CUDA device: the JK-CALS path has no CPU fallback")
    return torch


def column_major_flat(T):
    """Return (flat buffer, dims, is_device) with T's first index fastest (Eq. 3 layout)."""
    try:
        import torch
        if isinstance(T, torch.Tensor):
            dims = tuple(T.shape)
            t = T.to(torch.float64).permute(*reversed(range(T.dim()))).contiguous().reshape(-1)
            return t, dims, t.is_cuda
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(T, dtype=np.float64)
    dims = a.shape
    return np.ravel(a, order="F"), dims, False


class _Config(ctypes.Structure):
    """struct jkcals_config (include/jkcals.h)."""
    _fields_ = [("ndims", ctypes.c_int), ("dims", ctypes.c_void_p), ("nmodels", ctypes.c_int),
                ("ranks", ctypes.c_void_p), ("d", ctypes.c_int64), ("sub_begin", ctypes.c_int64),
                ("sub_end", ctypes.c_int64), ("spare", ctypes.c_int), ("prec", ctypes.c_int),
                ("hist_cap", ctypes.c_int), ("device", ctypes.c_int)]


class JKCals:
    """One shard [sub_begin, sub_end) of the I_1 leave-one-out submodels on one GPU.

    d > 1 selects delete-d jackknife: submodel p is then GROUP p, leaving
    out mode-0 rows [p d, min(p d + d, I_0)); sub_range indexes groups (default all
    ceil(I_0/d) of them).

    rank may be a sequence of ranks (R_0, R_1, ...): a multi-model pool (the paper's "All"
    experiment): submodel id s = m * ceil(I_0/d) + g is model m's group g,
    all fused into one multi-factor per mode; set_init then takes one factor list per model."""

    def __init__(self, T, rank, sub_range=None, device=None, stream=None, hist_cap=None,
                 precision=FP64, dims=None, d=1, spare=0):
        torch = _torch()
        self._torch = torch
        flat, tdims, is_dev = column_major_flat(T)
        if dims is not None:
            tdims = tuple(int(d) for d in dims)
        self.dims = tuple(int(d) for d in tdims)
        self.pool = not np.isscalar(rank)
        self.ranks = [int(r) for r in rank] if self.pool else [int(rank)]
        self.N, self.R = len(self.dims), max(self.ranks)
        self.nmodels = len(self.ranks)
        if device is None:
            device = flat.device.index if is_dev else torch.cuda.current_device()
        self.device = int(device)
        self.d = int(d)
        # d = 0: plain CALS (one model per id, nothing left out); d < 0 is rejected by the ABI
        self.ngroups = -(-self.dims[0] // self.d) if self.d >= 1 else (1 if self.d == 0 else 0)
        nall = self.nmodels * self.ngroups
        self.sub_begin, self.sub_end = (0, nall) if sub_range is None else map(int, sub_range)
        self.nsub = self.sub_end - self.sub_begin
        self.hist_cap = int(hist_cap or DEFAULT_MAX_ITERS)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        L = lib()
        d = _i64(self.dims)
        rk = np.ascontiguousarray(self.ranks, dtype=np.int32)
        self._cfg_keep = (d, rk)
        cfg = _Config(self.N, d.ctypes.data, self.nmodels, rk.ctypes.data, self.d, self.sub_begin, self.sub_end,
                      int(spare), int(precision), self.hist_cap, self.device)
        nbytes = L.jkcals_config_workspace_bytes(ctypes.byref(cfg))
        if nbytes == 0:
            raise JKCalsError(-1, f"unsupported arguments dims={self.dims} rank={self.R} nsub={self.nsub}")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._keep = flat
        tptr = flat.data_ptr() if is_dev else flat.ctypes.data
        h = ctypes.c_void_p()
        st = L.jkcals_create_config(ctypes.byref(h), ctypes.byref(cfg), ctypes.c_void_p(tptr), 1 if is_dev else 0,
                                    ctypes.c_void_p(self.stream.cuda_stream),
                                    ctypes.c_void_p(self.workspace.data_ptr()), nbytes)
        self._h = h
        if st != 0:
            msg = L.jkcals_last_error(h).decode() if h.value else ""
            self.close()
            raise JKCalsError(st, msg)
        self._keep = None  # the tensor now lives in the workspace
        self.nslots = L.jkcals_num_slots(h)

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st != 0:
            raise JKCalsError(st, lib().jkcals_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().jkcals_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI
    def set_init(self, P):
        """Warm start from the overall model P = [U_1..U_N] (Alg. 2 alg:jk:model_subsample); a
        pool takes [P_model0, P_model1, ...]."""
        models = P if self.pool else [P]
        if len(models) != self.nmodels:
            raise JKCalsError(-1, f"expected {self.nmodels} models, got {len(models)}")
        mats = []
        for mi, Pm in enumerate(models):
            for n, p in enumerate(Pm):
                m = np.asfortranarray(np.asarray(p, dtype=np.float64))
                if m.shape != (self.dims[n], self.ranks[mi]):
                    raise JKCalsError(-1, f"P[{mi}][{n}] has shape {m.shape}, expected "
                                          f"{(self.dims[n], self.ranks[mi])}")
                mats.append(m)
        self._init_keep = mats
        arr = (ctypes.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
        self._check(lib().jkcals_set_init(self._h, arr))

    def set_init_submodel(self, p, mode, U):
        m = np.asfortranarray(np.asarray(U, dtype=np.float64))
        self._check(lib().jkcals_set_init_submodel(self._h, int(p), int(mode), _p(m)))

    def set_init_all(self, mode, U_all):
        """Every submodel's mode-`mode` block at once, in the all_factors layout (array or list)."""
        parts = list(U_all) if not isinstance(U_all, np.ndarray) or U_all.ndim == 3 else [U_all]
        flat = np.concatenate([np.ravel(np.asarray(u, dtype=np.float64), order="F") for u in parts])
        self._check(lib().jkcals_set_init_all(self._h, int(mode), _p(flat)))

    def iterate(self, max_iters=DEFAULT_MAX_ITERS, tol=DEFAULT_TOL):
        done = ctypes.c_int()
        self._check(lib().jkcals_iterate(self._h, int(max_iters), float(tol), ctypes.byref(done)))
        return done.value

    def group_of(self, p):
        return p % self.ngroups

    def model_of(self, p):
        return p // self.ngroups

    def rank_of(self, p):
        return self.ranks[p // self.ngroups]

    def group_rows(self, p):
        """Mode-0 rows left out by submodel p (its group g = p mod ceil(I_0/d)); 0 for CALS."""
        g = p % self.ngroups
        return min(self.d, self.dims[0] - g * self.d)

    def factors(self, p):
        """Submodel p: ([U_0 ((I_0-|group|) x R, the group's rows dropped), U_1, ...], lambda)."""
        R = self.rank_of(p)
        out, lam = [], np.zeros(R)
        for n in range(self.N):
            rows = self.dims[n] - self.group_rows(p) if n == 0 else self.dims[n]
            U = np.zeros((rows, R), order="F")
            self._check(lib().jkcals_get_factors(self._h, int(p), n, _p(U), _p(lam) if n == self.N - 1 else None))
            out.append(U)
        return out, lam

    def all_factors(self, mode):
        """Every submodel's mode-`mode` factor at once: array (n_sub, rows, R) (the group's rows
        dropped in mode 0) and lambda (n_sub, R). With delete-d and a ragged last group the
        mode-0 factors come back as a list of (rows_q, R) arrays instead."""
        subs = [int(p) for p in self.ids() if p >= 0]   # owned submodels in slot order
        R_q = [self.rank_of(p) for p in subs]
        if mode == 0:
            rows_q = [self.dims[0] - self.group_rows(p) for p in subs]
        else:
            rows_q = [self.dims[mode]] * len(subs)
        flat = np.zeros(sum(r * c for r, c in zip(rows_q, R_q)))
        lamf = np.zeros(sum(R_q))
        self._check(lib().jkcals_get_all_factors(self._h, int(mode), _p(flat), _p(lamf)))
        if len(set(rows_q)) == 1 and len(set(R_q)) == 1:
            R = R_q[0]
            U = flat.reshape(len(subs), R, rows_q[0])  # per submodel a column-major rows x R
            return np.ascontiguousarray(U.transpose(0, 2, 1)), lamf.reshape(len(subs), R)
        out, lam, off, lo = [], [], 0, 0
        for r_, R in zip(rows_q, R_q):
            out.append(flat[off:off + r_ * R].reshape((r_, R), order="F"))
            lam.append(lamf[lo:lo + R])
            off += r_ * R
            lo += R
        return out, lam

    def block(self, p, mode):
        """Submodel p's full fused block of mode `mode` (mode 0 keeps the zero row p)."""
        U = np.zeros((self.dims[mode], self.rank_of(p)), order="F")
        self._check(lib().jkcals_get_block(self._h, int(p), int(mode), _p(U)))
        return U

    def status(self):
        n = self.nslots   # per slot (slot q holds ids()[q])
        fit, err = np.zeros(n), np.zeros(n)
        it, fl = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        self._check(lib().jkcals_get_status(self._h, _p(fit), _p(err), _p(it), _p(fl)))
        return {"fit": fit, "err": err, "iters": it, "flags": fl}

    def history(self, p, cap=None):
        cap = cap or self.hist_cap
        buf, cnt = np.zeros(cap), ctypes.c_int()
        self._check(lib().jkcals_get_history(self._h, int(p), _p(buf), cap, ctypes.byref(cnt)))
        return buf[: cnt.value]

    def jackknife_stats(self, mode, model=0):
        shp = (self.dims[mode], self.ranks[model])
        mean, std = np.zeros(shp, order="F"), np.zeros(shp, order="F")
        self._check(lib().jkcals_get_model_stats(self._h, int(model), int(mode), _p(mean), _p(std)))
        return mean, std

    def local_moments(self, mode, model=0):
        shp = (self.dims[mode], self.ranks[model])
        cnt, mean, m2 = (np.zeros(shp, order="F") for _ in range(3))
        self._check(lib().jkcals_get_model_moments(self._h, int(model), int(mode), _p(cnt), _p(mean), _p(m2)))
        return cnt, mean, m2

    # ------------------------------------------------------------------ slots / migration (NEXT #4)
    def ids(self):
        """Global submodel id held by each slot (-1 = free)."""
        out = np.zeros(self.nslots, dtype=np.int64)
        self._check(lib().jkcals_get_ids(self._h, _p(out)))
        return out

    def active_ids(self):
        """Ids of the owned submodels that still iterate (not converged, not failed)."""
        ids, fl = self.ids(), self.status()["flags"]
        return [int(p) for p, f in zip(ids, fl) if p >= 0 and not (f & 5)]

    def export_submodel(self, p):
        """Serialise submodel p's live ALS state (bytes) and remove it from this handle."""
        nb = lib().jkcals_state_bytes(self._h, int(p))
        if nb == 0:
            raise JKCalsError(-1, f"submodel {p} is not on this handle")
        buf = np.zeros(nb // 8)
        self._check(lib().jkcals_export_submodel(self._h, int(p), _p(buf), nb))
        return buf.tobytes()

    def import_submodel(self, state):
        """Adopt a submodel exported by another handle of the same problem (a free slot needed)."""
        buf = np.frombuffer(bytes(state), dtype=np.float64).copy()
        self._check(lib().jkcals_import_submodel(self._h, _p(buf), buf.nbytes))

    # ------------------------------------------------------------------ alignment (NEXT #3)
    def align(self):
        """Align every submodel to its model's warm start (Alg. 2 alg:jk:perm_scale)."""
        self._check(lib().jkcals_align(self._h))

    def alignment(self, p):
        R = self.rank_of(p)
        perm, sign, cong = np.zeros(R, dtype=np.int32), np.zeros((self.N, R), dtype=np.int32), np.zeros(R)
        self._check(lib().jkcals_get_alignment(self._h, int(p), _p(perm), _p(sign), _p(cong)))
        return perm, sign, cong

    def aligned_factors(self, p):
        R = self.rank_of(p)
        out = []
        for n in range(self.N):
            rows = self.dims[n] - self.group_rows(p) if n == 0 else self.dims[n]
            U = np.zeros((rows, R), order="F")
            self._check(lib().jkcals_get_aligned_factors(self._h, int(p), n, _p(U)))
            out.append(U)
        return out

    def aligned_moments(self, mode, model=0):
        shp = (self.dims[mode], self.ranks[model])
        cnt, mean, m2 = (np.zeros(shp, order="F") for _ in range(3))
        self._check(lib().jkcals_get_aligned_moments(self._h, int(model), int(mode), _p(cnt), _p(mean), _p(m2)))
        return cnt, mean, m2

    def aligned_stats(self, mode, model=0):
        shp = (self.dims[mode], self.ranks[model])
        mean, std = np.zeros(shp, order="F"), np.zeros(shp, order="F")
        self._check(lib().jkcals_get_aligned_stats(self._h, int(model), int(mode), _p(mean), _p(std)))
        return mean, std

    def set_instrument(self, on=True):
        self._check(lib().jkcals_set_instrument(self._h, 1 if on else 0))

    def kernel_times(self):
        a, b, n = np.zeros(self.N), np.zeros(self.N), ctypes.c_int64()
        self._check(lib().jkcals_get_kernel_times(self._h, _p(a), _p(b), ctypes.byref(n)))
        return a, b, n.value

    def sweep_flops(self):
        return lib().jkcals_sweep_flops(self._h)

    def launches_per_sweep(self):
        return lib().jkcals_launches_per_sweep(self._h)


def cals(T, ranks, inits=None, **kw):
    """Plain CALS (§3.3): len(ranks) CP models of T fitted concurrently in one
    fused sweep, each from its own initial model (nothing is left out: d = 0). Call
    set_init(inits) with one factor list per model (or pass inits here)."""
    h = JKCals(T, list(ranks), d=0, **kw)
    if inits is not None:
        h.set_init(inits)
    return h


# ---------------------------------------------------------------------- stand-alone ops
def mttkrp(T_flat, dims, n, U, C):
    """Fused MTTKRP on device tensors. T_flat: float64 cuda, column-major flat; U: list of
    row-major (dims[m], ldu) float64 cuda tensors (U[n] may be any placeholder).
    Returns M (dims[n], C) row-major torch tensor."""
    torch = _torch()
    L = lib()
    d = _i64(dims)
    ldu = U[(n + 1) % len(dims)].shape[1]
    dev = T_flat.device.index
    nb = L.jkcals_mttkrp_scratch_bytes(len(dims), _p(d), n, C, dev)
    if nb == 0:
        raise JKCalsError(-1, "unsupported mttkrp arguments")
    scratch = torch.empty(nb, dtype=torch.uint8, device=T_flat.device)
    M = torch.empty((dims[n], C), dtype=torch.float64, device=T_flat.device)
    ptrs = (ctypes.c_void_p * len(dims))(*[u.data_ptr() for u in U])
    st = L.jkcals_mttkrp(len(dims), _p(d), n, ctypes.c_void_p(T_flat.data_ptr()), ptrs, C, ldu,
                         ctypes.c_void_p(M.data_ptr()), C, ctypes.c_void_p(scratch.data_ptr()), nb,
                         ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != 0:
        raise JKCalsError(st, "jkcals_mttkrp failed")
    return M


def mttkrp_i8(T_flat, dims, n, U, C):
    """EXPERIMENTAL: the same MTTKRP, FP64-accurate from INT8 tcgen05 MMAs."""
    torch = _torch()
    L = lib()
    d = _i64(dims)
    ldu = U[(n + 1) % len(dims)].shape[1]
    dev = T_flat.device.index
    nb = L.jkcals_mttkrp_i8_scratch_bytes(len(dims), _p(d), n, C, dev)
    if nb == 0:
        raise JKCalsError(-1, "unsupported mttkrp_i8 arguments")
    scratch = torch.empty(nb, dtype=torch.uint8, device=T_flat.device)
    M = torch.empty((dims[n], C), dtype=torch.float64, device=T_flat.device)
    ptrs = (ctypes.c_void_p * len(dims))(*[u.data_ptr() for u in U])
    st = L.jkcals_mttkrp_i8(len(dims), _p(d), n, ctypes.c_void_p(T_flat.data_ptr()), ptrs, C, ldu,
                            ctypes.c_void_p(M.data_ptr()), C, ctypes.c_void_p(scratch.data_ptr()), nb,
                            ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != 0:
        raise JKCalsError(st, "jkcals_mttkrp_i8 failed")
    return M


def merge_moments(parts):
    """Fold per-shard (count, mean, M2) arrays in part order with the library's Chan merge
    (jkcals_merge_moments; host computation, no GPU needed). Returns (count, mean, M2)."""
    shape = np.shape(parts[0][1])
    cs, ms, ss = (np.ascontiguousarray(np.stack([np.ravel(np.asarray(p[i], dtype=np.float64), order="F")
                                                 for p in parts])) for i in range(3))
    n = cs.shape[1]
    c, m, s = np.zeros(n), np.zeros(n), np.zeros(n)
    st = lib().jkcals_merge_moments(len(parts), n, _p(cs), _p(ms), _p(ss), _p(c), _p(m), _p(s))
    if st != 0:
        raise JKCalsError(st, "jkcals_merge_moments failed")
    return tuple(np.reshape(x, shape, order="F") for x in (c, m, s))


def krp(dims, n, U, C, out=None):
    """Materialised Khatri-Rao product K (J_n, C) row-major on the device."""
    torch = _torch()
    d = _i64(dims)
    J = int(np.prod([dims[m] for m in range(len(dims)) if m != n]))
    ldu = U[(n + 1) % len(dims)].shape[1]
    dev = U[(n + 1) % len(dims)].device
    if out is None:
        out = torch.empty((J, C), dtype=torch.float64, device=dev)
    ptrs = (ctypes.c_void_p * len(dims))(*[u.data_ptr() for u in U])
    st = lib().jkcals_krp(len(dims), _p(d), n, ptrs, C, ldu, ctypes.c_void_p(out.data_ptr()), out.shape[1],
                          ctypes.c_void_p(torch.cuda.current_stream(dev.index).cuda_stream))
    if st != 0:
        raise JKCalsError(st, "jkcals_krp failed")
    return out
