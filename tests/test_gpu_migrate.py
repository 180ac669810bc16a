"""GPU tests for submodel migration between handles (tol-mode rebalancing).

Two handles in one process stand in for two ranks (the transport is torch.distributed in
production, covered by the gloo test in test_host.py). A migrated submodel must finish with the
same factors as without migration (rounding-level: the fused layout's split-K order changes)
and match the oracle at the usual 1e-10.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_pool, make_workload

pytestmark = pytest.mark.gpu
NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def local_balanced(hs, max_iters, tol, every):
    """iterate_balanced with an in-process transport (the plan and apply_moves of dist.py)."""
    from paper_2112_03985_b200.dist import apply_moves, plan_moves
    box = {}
    done = 0
    while done < max_iters:
        ran = [h.iterate(min(every, max_iters - done), tol) for h in hs]
        done += max(ran)
        act = [len(h.active_ids()) for h in hs]
        if sum(act) == 0:
            break
        free = [int((h.ids() < 0).sum()) for h in hs]
        moves = plan_moves(act, free)
        for r, h in enumerate(hs):      # sources first (their sends land in the box)
            apply_moves(h, [m for m in moves if m[0] == r], r,
                        lambda dst, b, r=r: box.setdefault((r, dst), []).append(b), None)
        for r, h in enumerate(hs):
            apply_moves(h, [m for m in moves if m[1] == r], r, None,
                        lambda src, r=r: box[(src, r)].pop(0))
    return done


def test_export_import_roundtrip_fixed_sweeps():
    # move submodels 3 and 7 from A to B after 10 sweeps, run 20 more: same result as the oracle
    from paper_2112_03985_b200 import JKCals
    w = make_workload("tiny")
    A = JKCals(w.T, w.R, sub_range=(0, 10), hist_cap=30, spare=2)
    B = JKCals(w.T, w.R, sub_range=(0, 1), hist_cap=30, spare=2)   # owns submodel 0 only
    A.set_init(w.P)
    B.set_init(w.P)
    A.iterate(10, 0.0)
    B.iterate(10, 0.0)
    for p in (3, 7):
        B.import_submodel(A.export_submodel(p))
    assert 3 not in A.ids() and 7 not in A.ids() and {3, 7} <= set(B.ids().tolist())
    A.iterate(20, 0.0)
    B.iterate(20, 0.0)
    res = O.jk_als(w.T, w.P, max_iters=30, nthreads=NCPU)
    for p in range(10):
        h = B if p in (3, 7) else A
        fac, lam = h.factors(p)
        for a, b in zip(fac, res.factors[p]):
            assert rel(a, b) <= 1e-10, (p, rel(a, b))
        hg = h.history(p)
        assert len(hg) == 30 and np.allclose(hg, res.history(p), rtol=1e-9)
        assert np.all(h.block(p, 0)[p] == 0.0)
    with pytest.raises(Exception):
        B.import_submodel(A.export_submodel(5))   # B has no free slot left


def test_rebalanced_tol_run_matches_oracle():
    # shard syn50 R3 over two "ranks" with tol; rebalance every 5 sweeps; all submodels must
    # end exactly as the oracle's (same iteration counts, factors within 1e-10)
    from paper_2112_03985_b200 import JKCals
    w = make_workload("syn50_r3")
    hs = [JKCals(w.T, w.R, sub_range=r, hist_cap=400, spare=25) for r in ((0, 25), (25, 50))]
    for h in hs:
        h.set_init(w.P)
    local_balanced(hs, 400, 1e-9, every=5)
    res = O.jk_als(w.T, w.P, max_iters=400, tol=1e-9, nthreads=NCPU)
    seen = set()
    for h in hs:
        st = h.status()
        for q, p in enumerate(h.ids()):
            if p < 0:
                continue
            seen.add(int(p))
            assert st["iters"][q] == res.iters[p], (p, st["iters"][q], res.iters[p])
            fac, _ = h.factors(int(p))
            for a, b in zip(fac, res.factors[p]):
                assert rel(a, b) <= 1e-10, (p, rel(a, b))
    assert seen == set(range(50))


def test_migrate_pool_mixed_ranks():
    from paper_2112_03985_b200 import JKCals
    w = make_pool(((16, 12, 8), (2, 4), 4, 0.01, "syn", 30), seed=7)
    A = JKCals(w.T, list(w.ranks), sub_range=(0, 32), hist_cap=30, spare=1)
    B = JKCals(w.T, list(w.ranks), sub_range=(0, 1), hist_cap=30, spare=3)
    A.set_init(w.Ps)
    B.set_init(w.Ps)
    A.iterate(12, 0.0)
    B.iterate(12, 0.0)
    for p in (5, 20, 31):                     # one rank-2 and two rank-4 submodels
        B.import_submodel(A.export_submodel(p))
    A.iterate(18, 0.0)
    B.iterate(18, 0.0)
    for m, P in enumerate(w.Ps):
        res = O.jk_als(w.T, P, max_iters=30, nthreads=NCPU)
        for g in range(16):
            p = m * 16 + g
            h = B if p in (5, 20, 31) else A
            fac, _ = h.factors(p)
            for a, b in zip(fac, res.factors[g]):
                assert rel(a, b) <= 1e-10, (p, rel(a, b))
