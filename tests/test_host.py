"""CPU-only tests of the host logic and the boundary (`-m "not gpu"`).

* the C-ABI library builds for sm_100a, loads, and exports every symbol include/jkcals.h declares;
* the product path has no CPU fallback (raises without a GPU);
* the flop model matches the numbers the paper prints (tests/golden/paper_flops.txt);
* shard planning and Chan moment merging; a world_size-2 gloo run of the end-of-run gathers.
"""
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "jkcals.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jkcals_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2112_03985_b200 import jkcals as J
    L = J.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(J.EXPORTED)
    out = subprocess.run(["nm", "-D", J._build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (jkcals_\w+)", out))
    assert set(syms) <= exported


def test_library_is_sm100a():
    from paper_2112_03985_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _build.LIB], capture_output=True,
                          text=True).stdout
    funcs = sass.split("Function : ")
    hot = [f for f in funcs if f.startswith("_ZN2jk18mttkrp_dmma_kernel")]
    # NT 1..8 x {n == 0, n >= 1} x {2, 4} stages x {128, 80}-column tiles x {16, 20}-deep k-tiles
    assert len(hot) == 128
    for f in hot:
        assert "DMMA" in f     # FP64 tensor-pipe instruction in the hot kernel
        assert "UTMALDG" in f  # TMA (cp.async.bulk.tensor) staging of the tensor tiles
        assert "UBLKCP" in f   # bulk copies of the Khatri-Rao factor rows


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2112_03985_b200 import JKCals, JKCalsError
    with pytest.raises(JKCalsError):
        JKCals(np.zeros((4, 3, 2)), 1)


def _golden():
    vals = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_flops.txt")):
        if line.strip() and not line.startswith("#"):
            name, value = line.split()[:2]
            vals[name] = int(value)
    return vals


def test_flop_model_matches_paper():
    from paper_2112_03985_b200.flops import jk_als_mttkrp_flops, jk_cals_mttkrp_flops, mttkrp_flops, overhead_ratio
    g = _golden()
    assert mttkrp_flops((50, 200, 200), 5) == g["mttkrp_flops_50x200x200_R5"]
    assert mttkrp_flops((50, 200, 200), 50 * 5) == g["fused_flops_50x200x200_K50_R5"]
    r = overhead_ratio((50, 30, 30), 5, d=1)
    assert (r.numerator, r.denominator) == (g["jk_ratio_num_I50_d1"], g["jk_ratio_den_I50_d1"])
    r10 = overhead_ratio((50, 30, 30), 5, d=10)
    assert r10 == 50 / 40 and r10 <= 2
    assert jk_cals_mttkrp_flops((50, 200, 200), 5) == 50 * mttkrp_flops((50, 200, 200), 5)
    assert jk_als_mttkrp_flops((50, 200, 200), 5) == 50 * mttkrp_flops((49, 200, 200), 5)
    # delete-d: d = I/2 is the worst case, ratio exactly 2
    assert overhead_ratio((50, 30, 30), 5, d=25) == 2
    # d does not divide I: ceil(I/d) groups, the last one smaller
    assert jk_cals_mttkrp_flops((10, 8, 6), 2, d=3) == 4 * mttkrp_flops((10, 8, 6), 2)
    assert jk_als_mttkrp_flops((10, 8, 6), 2, d=3) == 3 * mttkrp_flops((7, 8, 6), 2) + mttkrp_flops((9, 8, 6), 2)


def test_shard_partition():
    from paper_2112_03985_b200.dist import shard
    for I0 in (2, 7, 50, 200, 268):
        for G in (1, 2, 3, 4, 8):
            if G > I0:
                continue
            ranges = [shard(I0, G, g) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == I0
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and b > a
    assert [shard(200, 8, g) for g in range(8)][1] == (25, 50)


def test_chan_merge_exact():
    from paper_2112_03985_b200.dist import chan_merge, jackknife_std, merge_moments
    g = np.random.default_rng(0)
    X = g.standard_normal((11, 4, 3))

    def mom(Y):
        return np.full(Y.shape[1:], float(len(Y))), Y.mean(0), ((Y - Y.mean(0)) ** 2).sum(0)

    parts = [mom(X[:3]), mom(X[3:4]), mom(X[4:])]
    c, m, s = merge_moments(parts)
    c0, m0, s0 = mom(X)
    assert np.allclose(m, m0, rtol=1e-14) and np.allclose(s, s0, rtol=1e-12) and np.all(c == 11)
    assert np.allclose(jackknife_std(c, s), np.sqrt(10) * X.std(0), rtol=1e-12)
    c1, m1, s1 = chan_merge(np.zeros((4, 3)), np.zeros((4, 3)), np.zeros((4, 3)), *mom(X))
    assert np.allclose(m1, m0) and np.allclose(s1, s0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_GLOO_SCRIPT = r"""
import os, sys, numpy as np, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2112_03985_b200.dist import allgather_moments, allgather_vector, shard, jackknife_std
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=int(sys.argv[3]), world_size=2)
r = dist.get_rank()
X = np.random.default_rng(5).standard_normal((9, 4, 3))   # 9 "submodels" of a 4x3 factor
a, b = shard(9, 2, r)
Y = X[a:b]
loc = (np.full((4, 3), float(len(Y))), Y.mean(0), ((Y - Y.mean(0)) ** 2).sum(0))
c, m, s = allgather_moments(loc)
assert np.allclose(m, X.mean(0), rtol=1e-13) and np.allclose(jackknife_std(c, s), np.sqrt(8) * X.std(0), rtol=1e-12)
fits = allgather_vector(np.arange(a, b, dtype=float))
assert np.array_equal(fits, np.arange(9.0)), fits
dist.barrier()
dist.destroy_process_group()
print("ok", r)
"""


def test_gloo_world2_gathers(tmp_path):
    script = tmp_path / "g.py"
    script.write_text(_GLOO_SCRIPT)
    port = str(_free_port())
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, port, str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=180) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
        assert o.startswith("ok")


def test_plan_moves_balances_within_free_slots():
    from paper_2112_03985_b200.dist import plan_moves
    assert plan_moves([10, 2], [0, 6]) == [(0, 1, 4)]
    assert plan_moves([5, 5, 5], [2, 2, 2]) == []
    # capacity-bound: the destination only has 1 free slot
    assert plan_moves([9, 0], [0, 1]) == [(0, 1, 1)]
    # 4 ranks, one loaded: balanced to max - min <= 1 (free slots permitting)
    act, free = [12, 0, 0, 0], [0, 8, 8, 8]
    moves = plan_moves(act, free)
    for s, d, n in moves:
        act[s] -= n
        act[d] += n
    assert max(act) - min(act) <= 1 and sum(act) == 12
    assert plan_moves([3], [5]) == []


_GLOO_REBALANCE = r"""
import sys, numpy as np, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2112_03985_b200.dist import rebalance

class FakeHandle:
    # stands in for JKCals on CPU: slots with ids, an active set, opaque per-submodel states
    def __init__(self, ids, active, spare):
        self.slots = list(ids) + [-1] * spare
        self.act = set(active)
    def ids(self):
        return np.array(self.slots, dtype=np.int64)
    def active_ids(self):
        return sorted(p for p in self.slots if p >= 0 and p in self.act)
    def export_submodel(self, p):
        self.slots[self.slots.index(p)] = -1
        self.act.discard(p)
        return np.array([p, 7 * p], dtype=np.float64).tobytes()
    def import_submodel(self, b):
        p, chk = np.frombuffer(b, dtype=np.float64)
        assert chk == 7 * p
        self.slots[self.slots.index(-1)] = int(p)
        self.act.add(int(p))

dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=int(sys.argv[3]), world_size=2)
r = dist.get_rank()
# rank 0: 10 active of its 12; rank 1: 1 active of its 12 (the rest converged); 6 spare slots each
h = FakeHandle(range(12 * r, 12 * r + 12), range(12 * r, 12 * r + (10 if r == 0 else 1)), 6)
moves = rebalance(h)
assert moves == [(0, 1, 4)], moves
n = len(h.active_ids())
assert n == (6 if r == 0 else 5), (r, n, h.active_ids())
if r == 1:
    assert h.active_ids() == [6, 7, 8, 9, 12], h.active_ids()
dist.barrier()
dist.destroy_process_group()
print("ok", r)
"""


def test_gloo_world2_rebalance(tmp_path):
    script = tmp_path / "rb.py"
    script.write_text(_GLOO_REBALANCE)
    port = str(_free_port())
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, port, str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=180) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
        assert o.startswith("ok")


def test_binding_defaults_follow_the_paper():
    # tol 1e-6 and max_iters 1000
    from paper_2112_03985_b200 import DEFAULT_MAX_ITERS, DEFAULT_TOL
    assert DEFAULT_TOL == 1e-6 and DEFAULT_MAX_ITERS == 1000


def test_header_is_plain_c99_and_links(tmp_path):
    # include/jkcals.h compiles as C99 and a C program links against libjkcals.so (no GPU needed
    # to build; tests/test_gpu_robust.py runs the same program on a B200)
    import subprocess
    from paper_2112_03985_b200 import _build
    lib = _build.build()
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-O2",
                           os.path.join(ROOT, "tests", "c_abi_demo.c"), "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", "-L", os.path.dirname(lib), "-ljkcals",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", str(tmp_path / "demo")])
    assert (tmp_path / "demo").exists()
