"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no MTTKRP, no ALS, no
Gramians, no solves): it only draws random planted factors, composes the
planted tensor T = [[A_1..A_N]] + noise (the input recipe of SURVEY §8d /
SPEC.md:426) and a warm-start model P. See DESIGN.md "Input recipe".
"""
from .workloads import (CONFIGS, POOLS, PoolWorkload, Workload, make_pool, make_tensor,  # noqa: F401
                        make_warm_start, make_workload)
