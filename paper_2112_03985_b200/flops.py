"""The paper's flop model (host logic, no GPU).

* one MTTKRP costs 2 R prod_i I_i flops (§3.2);
* CALS fuses K models into one MTTKRP of width sum_i R_i (§3.3);
* JK-ALS MTTKRPs: (I/d) * 2R(I-d) prod_{i != n} I_i per mode; JK-CALS: 2 (I/d) R prod_i I_i
  per mode; ratio I/(I-d) <= 2 (§4.2).
"""
from __future__ import annotations

from fractions import Fraction
from math import prod


def mttkrp_flops(dims, width):
    """2 * width * prod(dims): one (fused) MTTKRP of the given column width."""
    return 2 * int(width) * prod(int(d) for d in dims)


def _groups(I, d):
    """Sizes of the ceil(I/d) contiguous delete-d groups (last smaller)."""
    return [min(d, I - g * d) for g in range(-(-I // d))]


def jk_cals_mttkrp_flops(dims, R, d=1, mode=0):
    """Fused JK-CALS MTTKRP flops of one mode; I/d -> ceil(I/d) groups."""
    I = int(dims[mode])
    return 2 * len(_groups(I, d)) * R * prod(int(x) for x in dims)


def jk_als_mttkrp_flops(dims, R, d=1, mode=0):
    """JK-ALS MTTKRP flops of one mode over all submodels: group g's submodel
    works on I - |g| slices."""
    I = int(dims[mode])
    rest = prod(int(x) for k, x in enumerate(dims) if k != mode)
    return sum(2 * R * (I - sz) * rest for sz in _groups(I, d))


def overhead_ratio(dims, R, d=1, mode=0):
    return Fraction(jk_cals_mttkrp_flops(dims, R, d, mode), jk_als_mttkrp_flops(dims, R, d, mode))
