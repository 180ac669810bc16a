"""Seeded synthetic workloads shaped like the paper's (BASELINE.json configs).

Recipe:
  * planted factors A_n: i.i.d. U(0,1) ("syn" kind), or fluorescence-like ("eem" kind:
    mode-0 lognormal concentrations, modes 1/2 non-negative Gaussian-bump spectra with a
    random centre and a width of 5-25 bins) -- samples x emission x excitation;
  * T = T0 + eta * ||T0|| / ||E|| * E, T0 = sum_r A_1(:,r) o ... o A_N(:,r), E ~ N(0,1);
  * warm start P ("an overall CP model fitted to T"): the planted factors
    (first R columns; extra U(0,1) columns if R > R_true) with 5 % Gaussian perturbation,
    so no ALS arithmetic is needed to produce it.
All arrays are float64; tensors are returned in column-major (Fortran) order, first
index fastest (Eq. 3). Random draws use numpy's PCG64 (default_rng).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# name -> (dims, R, R_true, eta, kind, sweeps)   (BASELINE.json "configs")
CONFIGS = {
    "tiny": ((10, 8, 6), 2, 2, 0.01, "syn", 50),
    "syn50_r1": ((50, 50, 50), 1, 5, 0.01, "syn", 100),
    "syn50_r2": ((50, 50, 50), 2, 5, 0.01, "syn", 100),
    "syn50_r3": ((50, 50, 50), 3, 5, 0.01, "syn", 100),
    "syn50_r4": ((50, 50, 50), 4, 5, 0.01, "syn", 100),
    "syn50_r5": ((50, 50, 50), 5, 5, 0.01, "syn", 100),
    "eem_r3": ((268, 201, 61), 3, 5, 0.02, "eem", 100),
    "eem_r4": ((268, 201, 61), 4, 5, 0.02, "eem", 100),
    "eem_r5": ((268, 201, 61), 5, 5, 0.02, "eem", 100),
    "eem_r6": ((268, 201, 61), 6, 5, 0.02, "eem", 100),
    "syn200": ((200, 200, 200), 5, 5, 0.01, "syn", 100),
    "4way": ((100, 60, 60, 30), 4, 4, 0.01, "syn", 100),
}


@dataclass
class Workload:
    name: str
    dims: tuple
    R: int
    sweeps: int
    T: np.ndarray          # float64, Fortran order, shape dims
    P: list                # warm start, list of (I_n, R) float64 Fortran arrays
    A: list                # planted factors (I_n, R_true)


def _planted_factors(rng, dims, R_true, kind):
    A = []
    for n, I in enumerate(dims):
        if kind == "eem" and n == 0:
            A.append(rng.lognormal(mean=0.0, sigma=1.0, size=(I, R_true)))
        elif kind == "eem":
            x = np.arange(I, dtype=np.float64)[:, None]
            mu = rng.uniform(0, I, size=(1, R_true))
            sig = rng.uniform(5, 25, size=(1, R_true))
            A.append(np.exp(-0.5 * ((x - mu) / sig) ** 2))
        else:
            A.append(rng.uniform(0.0, 1.0, size=(I, R_true)))
    return [np.asfortranarray(a) for a in A]


def compose(A):
    """T0 = sum_r A_0(:,r) o A_1(:,r) o ... (input composition only)."""
    R = A[0].shape[1]
    T = np.zeros(tuple(a.shape[0] for a in A), dtype=np.float64)
    for r in range(R):
        t = A[0][:, r]
        for a in A[1:]:
            t = np.multiply.outer(t, a[:, r])
        T += t
    return np.asfortranarray(T)


def make_tensor(dims, R_true, eta, kind="syn", seed=0):
    rng = np.random.default_rng(seed)
    A = _planted_factors(rng, dims, R_true, kind)
    T0 = compose(A)
    if eta > 0:
        E = rng.standard_normal(size=T0.shape)
        T = T0 + eta * np.linalg.norm(T0.ravel()) / np.linalg.norm(E.ravel()) * E
    else:
        T = T0
    return np.asfortranarray(T), A


def make_warm_start(A, R, seed=0, perturb=0.05):
    rng = np.random.default_rng(seed + 1000003)
    P = []
    for a in A:
        I, Rt = a.shape
        if R <= Rt:
            b = a[:, :R].copy()
        else:
            b = np.concatenate([a, rng.uniform(0.0, 1.0, size=(I, R - Rt))], axis=1)
        scale = np.abs(b).mean() if b.size else 1.0
        b = b + perturb * scale * rng.standard_normal(size=b.shape)
        P.append(np.asfortranarray(b))
    return P


def make_workload(name_or_spec, seed=0, sweeps=None) -> Workload:
    if isinstance(name_or_spec, str):
        dims, R, R_true, eta, kind, sw = CONFIGS[name_or_spec]
        name = name_or_spec
    else:
        dims, R, R_true, eta, kind, sw = name_or_spec
        name = "custom"
    T, A = make_tensor(dims, R_true, eta, kind, seed)
    P = make_warm_start(A, R, seed)
    return Workload(name, tuple(dims), R, sweeps if sweeps is not None else sw, T, P, A)


# Multi-model pools (the paper's "All" experiment; Fig. 5's {4,5,6} models,
# PAPER.md:590-593): name -> (dims, ranks, R_true, eta, kind, sweeps). Every model is warm-started
# from the planted factors of the SAME tensor (make_warm_start per rank).
POOLS = {
    "all_small": ((50, 100, 100), (3, 5, 7, 9), 5, 0.01, "syn", 100),
    "all_medium": ((50, 200, 200), (3, 5, 7, 9), 5, 0.01, "syn", 100),
    "eem_all": ((268, 201, 61), (4, 5, 6), 5, 0.02, "eem", 100),
}


@dataclass
class PoolWorkload:
    name: str
    dims: tuple
    ranks: tuple
    sweeps: int
    T: np.ndarray
    Ps: list               # one warm start (list of (I_n, R_m) arrays) per model
    A: list


def make_pool(name_or_spec, seed=0, sweeps=None) -> PoolWorkload:
    if isinstance(name_or_spec, str):
        dims, ranks, R_true, eta, kind, sw = POOLS[name_or_spec]
        name = name_or_spec
    else:
        dims, ranks, R_true, eta, kind, sw = name_or_spec
        name = "custom"
    T, A = make_tensor(dims, R_true, eta, kind, seed)
    Ps = [make_warm_start(A, R, seed) for R in ranks]
    return PoolWorkload(name, tuple(dims), tuple(ranks), sweeps if sweeps is not None else sw, T, Ps, A)
