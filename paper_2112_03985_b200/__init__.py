"""B200-native JK-CALS: concurrent ALS fitting of all leave-one-out CP submodels
(Psarras et al., arXiv 2112.03985, Alg. 3) in hand-written CUDA for sm_100a.

The compute path is libjkcals.so (C ABI: include/jkcals.h); this package only marshals
arguments (jkcals.py), plans shards and merges statistics across ranks (dist.py), and
counts the paper's flops (flops.py).
"""
from .flops import jk_als_mttkrp_flops, jk_cals_mttkrp_flops, mttkrp_flops  # noqa: F401
from .jkcals import (DEFAULT_MAX_ITERS, DEFAULT_TOL, JKCals, JKCalsError, cals, krp, lib,  # noqa: F401
                     mttkrp)
