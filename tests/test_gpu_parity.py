"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (BASELINE.json north_star): FP64 factors within 1e-10 relative Frobenius of the oracle
from identical initial factors and a fixed sweep count. The per-sweep error is compared with
|e_gpu - e_orc| <= 1e-9 |e_orc| + 1e-13 ||T_-p||^2 (e is a difference
of O(||T||^2) terms, so its absolute rounding is O(eps ||T||^2)).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_workload

pytestmark = pytest.mark.gpu

FTOL = 1e-10
NCPU = os.cpu_count() or 1


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def run_gpu(w, sweeps, tol=0.0, sub_range=None, hist_cap=None, instrument=False):
    from paper_2112_03985_b200 import JKCals
    h = JKCals(w.T, w.R, sub_range=sub_range, hist_cap=hist_cap or max(sweeps, 1))
    h.set_init(w.P)
    if instrument:
        h.set_instrument(True)
    done = h.iterate(sweeps, tol)
    return h, done


def check_against_oracle(h, res, p_list, nt2p=None):
    st = h.status()
    for q, p in enumerate(p_list):
        fac, lam = h.factors(p)
        for n, (a, b) in enumerate(zip(fac, res.factors[q])):
            assert rel(a, b) <= FTOL, (p, n, rel(a, b))
        assert rel(lam, res.lam[q]) <= FTOL, (p, rel(lam, res.lam[q]))
        hg, ho = h.history(p), res.history(q)
        assert len(hg) == len(ho) == res.iters[q]
        scale = nt2p[p] if nt2p is not None else abs(ho).max()
        assert np.all(np.abs(hg - ho) <= 1e-9 * np.abs(ho) + 1e-13 * scale), (p, np.abs(hg - ho).max())
        sub = p - h.sub_begin
        assert st["iters"][sub] == res.iters[q]
        assert (st["flags"][sub] & ~1) == (res.flags[q] & ~1), (p, st["flags"][sub], res.flags[q])
        # padded-row invariant: row p of the mode-0 block is exactly zero
        blk = h.block(p, 0)
        assert np.all(blk[p] == 0.0)


def nt2p_of(T):
    n2 = O.norm_sq(T)
    return n2 - O.slice_norms_sq(T, 0)


# ---------------------------------------------------------------- kernel-level parity
MTTKRP_CASES = [
    ((10, 8, 6), 20), ((50, 50, 50), 50), ((50, 50, 50), 250), ((37, 23, 11), 129),
    ((13, 7, 5, 3), 70), ((268, 30, 9), 33), ((5, 300, 4), 10), ((3, 2, 2), 1), ((17, 3, 4, 2, 3), 24),
]


@pytest.mark.parametrize("dims,C", MTTKRP_CASES)
def test_mttkrp_kernel_vs_oracle(dims, C):
    import torch
    from paper_2112_03985_b200 import mttkrp
    g = np.random.default_rng(sum(dims) + C)
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = []
    for u in U:
        pad = np.zeros((u.shape[0], ldu))
        pad[:, :C] = u
        Ud.append(torch.from_numpy(pad).cuda())
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(len(dims)):
        M = mttkrp(Td, dims, n, Ud, C).cpu().numpy()
        ref = O.mttkrp(T, U, n)
        scale = np.abs(ref).max()
        assert np.allclose(M, ref, rtol=1e-12, atol=1e-12 * scale), (dims, C, n, np.abs(M - ref).max() / scale)


def test_krp_kernel_vs_khatri_rao():
    import torch
    from paper_2112_03985_b200 import krp
    g = np.random.default_rng(3)
    dims, C = (7, 6, 5, 4), 13
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = 16
    Ud = []
    for u in U:
        pad = np.zeros((u.shape[0], ldu))
        pad[:, :C] = u
        Ud.append(torch.from_numpy(pad).cuda())
    for n in range(4):
        K = krp(dims, n, Ud, C).cpu().numpy()
        rest = [m for m in range(4) if m != n]
        ref = U[rest[0]]
        for m in rest[1:]:
            ref = O.khatri_rao(U[m], ref)  # descending KRP, earliest mode fastest (Eq. 1/3)
        assert np.array_equal(K, ref) or np.allclose(K, ref, rtol=1e-15, atol=0)


def test_krp_kernel_full_size_vector_path():
    # the materialised KRP at a realistic size (50 x 200 x 200, C = 96: the 4-wide vector path,
    # ldu % 4 == 0, and the register-cached slow-row product), every mode, bitwise vs the oracle's
    # Khatri-Rao (same multiplication order) -- or to 1 ulp if the compiler contracts differently
    import torch
    from paper_2112_03985_b200 import krp
    g = np.random.default_rng(11)
    dims, C, ldu = (50, 200, 200), 96, 128
    U = [g.standard_normal((I, C)) for I in dims]
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    for n in range(3):
        K = krp(dims, n, Ud, C).cpu().numpy()
        rest = [m for m in range(3) if m != n]
        ref = O.khatri_rao(U[rest[1]], U[rest[0]])
        assert K.shape == ref.shape
        assert np.allclose(K, ref, rtol=2.3e-16, atol=0), n


# ---------------------------------------------------------------- JK-CALS vs JK-ALS
def test_tiny_all_submodels():
    w = make_workload("tiny")
    h, done = run_gpu(w, w.sweeps)
    assert done == w.sweeps
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, range(10), nt2p_of(w.T))


@pytest.mark.parametrize("R", [1, 2, 3, 4, 5])
def test_syn50_all_submodels(R):
    w = make_workload(f"syn50_r{R}")
    h, _ = run_gpu(w, w.sweeps)
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, range(50), nt2p_of(w.T))


def test_edge_two_samples_rank1():
    w = make_workload(((2, 3, 4), 1, 1, 0.05, "syn", 30), seed=2)
    h, _ = run_gpu(w, 30)
    res = O.jk_als(w.T, w.P, max_iters=30)
    check_against_oracle(h, res, range(2), nt2p_of(w.T))


def test_edge_five_way_ragged():
    w = make_workload(((9, 5, 3, 4, 2), 3, 3, 0.02, "syn", 25), seed=4)
    h, _ = run_gpu(w, 25)
    res = O.jk_als(w.T, w.P, max_iters=25, nthreads=NCPU)
    check_against_oracle(h, res, range(9), nt2p_of(w.T))


def test_sampled_large_configs_4way():
    w = make_workload("4way")
    h, _ = run_gpu(w, w.sweeps)
    ps = [0, 1, 50, 99]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, ps, nt2p_of(w.T))


@pytest.mark.parametrize("name", ["eem_r3", "eem_r5"])
def test_sampled_eem(name):
    w = make_workload(name)
    h, _ = run_gpu(w, w.sweeps)
    ps = [0, 133, 267]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, ps, nt2p_of(w.T))


@pytest.mark.parametrize("name", ["eem_r4", "eem_r6"])
def test_sampled_eem_r4_r6_reported(name):
    # eem_r6 over-factors the rank-5 truth (A17: ALS can be degenerate there). r01
    # measured 4e-14 (r4) and 4e-12 (r6) after 100 sweeps, so both are held to the 1e-10 gate.
    w = make_workload(name)
    h, _ = run_gpu(w, w.sweeps)
    ps = [0, 200]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    worst = 0.0
    for q, p in enumerate(ps):
        for a, b in zip(h.factors(p)[0], res.factors[q]):
            worst = max(worst, rel(a, b))
    print(f"{name}: worst relative factor deviation vs oracle {worst:.3e}")
    assert worst <= FTOL, worst


def test_sampled_syn200_bench_config():
    w = make_workload("syn200")
    h, _ = run_gpu(w, w.sweeps)
    ps = [0, 1, 100, 199]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, ps, nt2p_of(w.T))


def test_small_shard_pre_reduced_pieces():
    # a syn200 shard at G = 8 (25 submodels, C = 125): one 128-column tile split ~59 ways, so the
    # stream-K pieces go through the warp-split reduce_pieces_kernel before the epilogue (the
    # r02 rewrite) -- sampled submodels of two shards against the oracle at the FP64 bar
    w = make_workload("syn200")
    for lo, hi, ps in ((0, 25, [0, 13, 24]), (175, 200, [175, 199])):
        h, _ = run_gpu(w, w.sweeps, sub_range=(lo, hi))
        res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
        check_against_oracle(h, res, ps, nt2p_of(w.T))
        h.close()


# ---------------------------------------------------------------- modes of operation
def test_tolerance_mode_and_compaction():
    w = make_workload("syn50_r3")
    h, done = run_gpu(w, 1000, tol=1e-6, hist_cap=1000)
    res = O.jk_als(w.T, w.P, max_iters=1000, tol=1e-6, nthreads=NCPU)
    assert done <= 1000
    assert len(set(res.iters.tolist())) > 1  # submodels converge at different sweeps
    check_against_oracle(h, res, range(50), nt2p_of(w.T))


def test_tol_device_trigger_equals_host_loop(monkeypatch):
    # tolerance mode runs as a CUDA-graph WHILE loop whose condition a device kernel sets (no host
    # round trip per sweep; the host wakes only to compact). The instrumented path checks on the
    # host after every sweep; both must stop at the same sweep with bit-identical factors, across
    # several compactions (syn50 R3: 64 fused columns converge -> compact).
    from paper_2112_03985_b200.jkcals import lib
    monkeypatch.setenv("JKCALS_RESIDENT", "0")
    w = make_workload("syn50_r3")
    h1, d1 = run_gpu(w, 1000, tol=1e-6, hist_cap=1000)
    assert "conditional graph" not in lib().jkcals_last_error(h1._h).decode()
    h2, d2 = run_gpu(w, 1000, tol=1e-6, hist_cap=1000, instrument=True)
    assert d1 == d2
    s1, s2 = h1.status(), h2.status()
    assert np.array_equal(s1["iters"], s2["iters"]) and np.array_equal(s1["flags"], s2["flags"])
    for p in range(50):
        for a, b in zip(h1.factors(p)[0], h2.factors(p)[0]):
            assert np.array_equal(a, b), p
    # a sweep budget that ends mid-run is honoured exactly
    h3, d3 = run_gpu(w, 7, tol=1e-6, hist_cap=1000)
    assert d3 == 7 and np.all(h3.status()["iters"] <= 7)


def test_shards_equal_full_and_merge():
    from paper_2112_03985_b200.dist import jackknife_std, merge_moments
    w = make_workload("syn50_r2")
    full, _ = run_gpu(w, 40)
    a, _ = run_gpu(w, 40, sub_range=(0, 20))
    b, _ = run_gpu(w, 40, sub_range=(20, 50))
    for p in range(50):
        src = a if p < 20 else b
        for x, y in zip(src.factors(p)[0], full.factors(p)[0]):
            assert rel(x, y) <= 1e-13
    for mode in (1, 2):
        mean, std = full.jackknife_stats(mode)
        c, m, s = merge_moments([a.local_moments(mode), b.local_moments(mode)])
        assert np.allclose(m, mean, rtol=1e-13, atol=1e-15)
        assert np.allclose(jackknife_std(c, s), std, rtol=1e-10, atol=1e-15)


def test_all_factors_equals_per_submodel():
    w = make_workload("tiny")
    h, _ = run_gpu(w, 12)
    for mode in range(3):
        U_all, lam_all = h.all_factors(mode)
        for p in range(10):
            fac, lam = h.factors(p)
            assert np.array_equal(U_all[p], fac[mode])
            assert np.array_equal(lam_all[p], lam)


def test_jackknife_stats_vs_oracle():
    w = make_workload("tiny")
    h, _ = run_gpu(w, w.sweeps)
    res = O.jk_als(w.T, w.P, max_iters=w.sweeps, nthreads=NCPU)
    for mode in (1, 2):
        X = np.stack([res.factors[q][mode] for q in range(10)])
        m_o, s_o = O.jackknife_stats(X)
        m_g, s_g = h.jackknife_stats(mode)
        assert rel(m_g, m_o) <= FTOL and rel(s_g, s_o) <= 1e-8


def test_pinv_fallback_is_per_submodel():
    # a zero column in one submodel's mode-1 init makes its H singular; only
    # that submodel takes the pseudoinverse path, and it still matches the oracle.
    from paper_2112_03985_b200 import JKCals
    w = make_workload("tiny")
    h = JKCals(w.T, w.R, hist_cap=20)
    h.set_init(w.P)
    bad = w.P[1].copy()
    bad[:, 1] = 0.0
    h.set_init_submodel(3, 1, bad)
    h.iterate(20, 0.0)
    st = h.status()
    assert st["flags"][3] & 2 and not np.any(np.delete(st["flags"], 3) & 2)
    res = O.jk_als(w.T, w.P, p_list=[0, 5], max_iters=20)
    check_against_oracle(h, res, [0, 5])
    Pb = [w.P[0], bad, w.P[2]]
    res3 = O.jk_als(w.T, Pb, p_list=[3], max_iters=20)
    assert res3.flags[0] & 2
    fac, _ = h.factors(3)
    for a, b in zip(fac, res3.factors[0]):
        assert rel(a, b) <= 1e-9


def test_deterministic_and_graph_equals_eager(monkeypatch):
    monkeypatch.setenv("JKCALS_RESIDENT", "0")  # the streamed path (graph replay vs eager launches)
    w = make_workload("syn50_r2")
    h1, _ = run_gpu(w, 15)
    h2, _ = run_gpu(w, 15)
    h3, _ = run_gpu(w, 15, instrument=True)
    for p in (0, 17, 49):
        for a, b, c in zip(h1.factors(p)[0], h2.factors(p)[0], h3.factors(p)[0]):
            assert np.array_equal(a, b) and np.array_equal(a, c)
    t_m, t_e, launches = h3.kernel_times()
    assert launches == 15 * 3 and np.all(t_m > 0) and np.all(t_e > 0)


def test_abi_errors():
    from paper_2112_03985_b200 import JKCals, JKCalsError
    w = make_workload("tiny")
    h = JKCals(w.T, 2)
    with pytest.raises(JKCalsError):
        h.iterate(1, 0.0)  # before set_init -> E_STATE
    with pytest.raises(JKCalsError):
        h.set_init([np.full((10, 2), np.nan), w.P[1], w.P[2]])
    with pytest.raises(JKCalsError):
        JKCals(np.full((3, 3, 3), np.inf), 1)
    with pytest.raises(JKCalsError):
        JKCals(w.T, 2, sub_range=(4, 11))


# ---------------------------------------------------------------- FP32 path (3xTF32 tcgen05)
FTOL32 = 1e-4  # north_star: the FP32 path matches the FP64 oracle to 1e-4 relative Frobenius


def run_gpu32(w, sweeps, sub_range=None):
    from paper_2112_03985_b200 import JKCals
    from paper_2112_03985_b200.jkcals import FP32
    h = JKCals(w.T, w.R, sub_range=sub_range, hist_cap=max(sweeps, 1), precision=FP32)
    h.set_init(w.P)
    h.iterate(sweeps, 0.0)
    return h


def check32(h, res, p_list):
    worst = 0.0
    for q, p in enumerate(p_list):
        fac, lam = h.factors(p)
        for a, b in zip(fac, res.factors[q]):
            worst = max(worst, rel(a, b))
        worst = max(worst, rel(lam, res.lam[q]))
        assert np.all(h.block(p, 0)[p] == 0.0)
    assert worst <= FTOL32, worst
    return worst


@pytest.mark.parametrize("name,ps", [("tiny", None), ("syn50_r5", None), ("4way", [0, 1, 50, 99])])
def test_fp32_path_vs_oracle(name, ps):
    w = make_workload(name)
    sweeps = min(w.sweeps, 50) if name == "4way" else w.sweeps
    h = run_gpu32(w, sweeps)
    p_list = list(range(w.dims[0])) if ps is None else ps
    res = O.jk_als(w.T, w.P, p_list=p_list, max_iters=sweeps, nthreads=NCPU)
    check32(h, res, p_list)


def test_fp32_fluorescence_shaped_full_config():
    # the eem R5 config (268 x 201 x 61, long contractions, fluorescence-shaped data): the FP32
    # accumulation chain length decides this one -- 768-product chains left 2.2e-4 (> the 1e-4
    # bar), 128-product chains 1.7e-5 at full size (profiles/r02_full_parity.jsonl) -- sampled
    # submodels after 100 sweeps
    w = make_workload("eem_r5")
    h = run_gpu32(w, w.sweeps)
    ps = [0, 100, 200, 267]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check32(h, res, ps)


def test_fp32_path_is_deterministic():
    # the FP32 drain adds each accumulation chain into the FP64 piece with bulk f64 adds; chains of
    # one piece are issued only after the previous chain's group completed, so two runs agree bitwise
    w = make_workload("syn50_r5")
    a = run_gpu32(w, 10)
    b = run_gpu32(w, 10)
    for p in (0, 7, 49):
        for x, y in zip(a.factors(p)[0], b.factors(p)[0]):
            assert np.array_equal(x, y), p


def test_fp32_pair_odd_tiles_and_one_cta_variant():
    # the CTA-pair (cta_group::2) FP32 kernel with an odd number of 128-column tiles (C = 60 x 6 =
    # 360: 3 tiles, the last super tile's second half dead) and a ragged I_n = 44, against the oracle;
    # the one-CTA kernel (JKCALS_TF32_PAIR=0, read once per process: subprocess) meets the same bar.
    # (R = R_true: an over-factored R = 6 > 5 model is ill-conditioned enough that BOTH FP32 kernels
    # land near 1e-3 -- tools/pair_diag.py -- a property of FP32, not of the kernel)
    import subprocess, sys
    spec = ((60, 44, 36), 6, 6, 0.01, "syn", 30)
    w = make_workload(spec)
    h = run_gpu32(w, w.sweeps)
    ps = [0, 31, 59]
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check32(h, res, ps)
    code = ("import numpy as np\n"
            "from synth import make_workload\n"
            "from paper_2112_03985_b200 import JKCals\n"
            f"w = make_workload({spec!r})\n"
            "h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=1)\n"
            "h.set_init(w.P); h.iterate(w.sweeps, 0.0)\n"
            "np.save('/tmp/jk_onecta.npy', np.concatenate([np.ravel(f) for p in (0, 31, 59) for f in h.factors(p)[0]]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, JKCALS_TF32_PAIR="0"), timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    one = np.load("/tmp/jk_onecta.npy")
    pair = np.concatenate([np.ravel(f) for p in ps for f in h.factors(p)[0]])
    assert rel(pair, one) <= FTOL32


@pytest.mark.parametrize("name,ps,max_iters", [("syn50_r3", None, 1000), ("4way", [0, 57], 60)])
def test_fp32_tol_mode_vs_oracle(name, ps, max_iters):
    """FP32 path in tol mode (the paper's tol = 1e-6): the last mode runs on the
    FP64 kernel (reading A24), so the error history is FP64-accurate for the FP32-path model and
    the stop decisions match the FP64 oracle's; factors within the FP32 bar."""
    from paper_2112_03985_b200 import JKCals
    from paper_2112_03985_b200.jkcals import FP32
    w = make_workload(name)
    p_list = list(range(w.dims[0])) if ps is None else ps
    h = JKCals(w.T, w.R, hist_cap=max_iters, precision=FP32)
    h.set_init(w.P)
    h.iterate(max_iters, 1e-6)
    res = O.jk_als(w.T, w.P, p_list=p_list, max_iters=max_iters, tol=1e-6, nthreads=NCPU)
    st = h.status()
    same = 0
    for q, p in enumerate(p_list):
        it_g, it_o = int(st["iters"][p]), int(res.iters[q])
        assert abs(it_g - it_o) <= 1, (p, it_g, it_o)  # the stop rule may flip at the threshold
        same += it_g == it_o
        hg, ho = h.history(p), res.history(q)
        k = min(len(hg), len(ho))
        # FP64-accurate errors of a model that is FP32-close to the oracle's (r01, all-FP32: 31 %)
        assert np.all(np.abs(hg[:k] - ho[:k]) <= 1e-3 * np.abs(ho[:k])), (p, np.abs(hg[:k] / ho[:k] - 1).max())
        if it_g == it_o:
            fac, lam = h.factors(p)
            for a_, b_ in zip(fac, res.factors[q]):
                assert rel(a_, b_) <= FTOL32, (p, rel(a_, b_))
    assert same >= 0.9 * len(p_list), (same, len(p_list))
    if ps is None:
        assert len(set(res.iters.tolist())) > 1


@pytest.mark.parametrize("dims,C", [((10, 8, 6), 20), ((37, 23, 11), 129), ((13, 7, 5, 3), 70),
                                    ((50, 50, 50), 250), ((5, 300, 4), 10),
                                    # I_q0 = 90 / 70 / 96 end inside the first half of the last K64 step
                                    # (its second K32 sub-step is skipped), 97 just past it
                                    ((90, 70, 9), 140), ((97, 96, 5), 64)])
def test_experimental_int8_sliced_mttkrp(dims, C):
    # the FP64-accurate MTTKRP from INT8 tcgen05 MMAs (7-digit slicing, exact int32
    # diagonal accumulators, S applied in FP64) matches the oracle like the DMMA kernel does
    import torch
    from paper_2112_03985_b200.jkcals import mttkrp_i8
    g = np.random.default_rng(sum(dims) + C + 7)
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(len(dims)):
        M = mttkrp_i8(Td, dims, n, Ud, C).cpu().numpy()
        ref = O.mttkrp(T, U, n)
        assert rel(M, ref) <= 1e-13, (dims, C, n, rel(M, ref))


def _spiky_tensor(g, dims):
    """Wide dynamic range: rows of T_(0) scaled over 1e-12 .. 1 and isolated spikes of
    1e4 .. 1e8 times their neighbours -- the scatter-like outliers of fluorescence data."""
    T = g.standard_normal(dims)
    T *= (10.0 ** g.uniform(-12, 0, dims[0])).reshape((-1,) + (1,) * (len(dims) - 1))
    flat = T.reshape(-1)
    for amp in (1e4, 1e6, 1e8):
        idx = g.choice(flat.size, 3, replace=False)
        flat[idx] *= amp
    return np.asfortranarray(T)


@pytest.mark.parametrize("dims,C", [((40, 30, 20), 64), ((13, 9, 7, 5), 40)])
def test_int8_sliced_mttkrp_wide_dynamic_range(dims, C):
    """FP64_I8 with per-(row, j') slab scaling of T: every row's MTTKRP matches the oracle to FP64
    accuracy relative to that row's own magnitude, spikes and 1e-12-scaled rows included."""
    import torch
    from paper_2112_03985_b200.jkcals import mttkrp_i8
    g = np.random.default_rng(11 + sum(dims))
    T = _spiky_tensor(g, dims)
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(len(dims)):
        M = mttkrp_i8(Td, dims, n, Ud, C).cpu().numpy()
        ref = O.mttkrp(T, U, n)
        absU = [np.abs(u) for u in U]
        absref = O.mttkrp(np.abs(T), absU, n)
        # the documented bound (include/jkcals.h): 49-bit digits relative to each (row i, j') slab's
        # largest |T| and each U_q0 column's largest |U| -> per slab normwise. Tb replaces every
        # entry of a slab (the contraction axis q0) by the slab's max |T|.
        q0 = 1 if n == 0 else 0
        Tb = np.broadcast_to(np.abs(T).max(axis=q0, keepdims=True), T.shape)
        bound = 2.0 ** -44 * O.mttkrp(np.asfortranarray(Tb), absU, n) + 1e-14 * absref
        assert np.all(np.abs(M - ref) <= bound), (dims, n, (np.abs(M - ref) / bound).max())
        # and relative to each element's own |T| x |KRP| magnitude it stays far below the FP64 parity
        # bar even with 1e8 spikes and rows scaled down to 1e-12 (r01's per-row scaling: ~1e-8)
        assert (np.abs(M - ref) / np.maximum(absref, 1e-300)).max() <= 1e-9


@pytest.mark.parametrize("spike", [None, 1e5])
def test_int8_sliced_fp64_path_wide_dynamic_range(spike):
    """The whole FP64_I8 JK-CALS loop on a tensor whose mode-0 slices span 1e-8 .. 1 is held to the
    FP64 bar (the per-(row, j') scales absorb any row scaling exactly). With a scatter-like 1e5 spike
    the per-slab normwise bound shows: the spike's slab keeps ~32 of 49 bits, so the FP64_I8 factors
    drift to ~1e-9 while the DMMA path stays at the bar -- the documented contract (include/jkcals.h)
    that keeps FP64_I8 supplementary."""
    from paper_2112_03985_b200 import JKCals
    g = np.random.default_rng(5)
    dims, R = (24, 18, 14), 3
    A = [g.uniform(0, 1, (I, R)) for I in dims]
    A[0] *= (10.0 ** g.uniform(-8, 0, dims[0]))[:, None]  # samples of very different magnitude
    T = np.einsum("ir,jr,kr->ijk", *A)
    T = T * (1 + 0.01 * g.standard_normal(dims))
    if spike:
        T[g.integers(0, 24), g.integers(0, 18), g.integers(0, 14)] *= spike
    T = np.asfortranarray(T)
    P = [np.asfortranarray(a + 0.05 * g.standard_normal(a.shape)) for a in A]
    res = O.jk_als(T, P, max_iters=30, nthreads=NCPU)
    worst = {}
    for prec in (0, 2):
        h = JKCals(T, R, hist_cap=30, precision=prec)
        h.set_init(P)
        h.iterate(30, 0.0)
        w_ = 0.0
        for p in range(dims[0]):
            fac, lam = h.factors(p)
            for a_, b_ in zip(fac, res.factors[p]):
                w_ = max(w_, rel(a_, b_))
        worst[prec] = w_
    assert worst[0] <= FTOL, worst
    assert worst[2] <= (FTOL if spike is None else 1e-7), worst


def test_int8_nonfinite_column_propagates():
    """A non-finite U_q0 entry reaches M as NaN (it used to be sliced into finite digits)."""
    import torch
    from paper_2112_03985_b200.jkcals import mttkrp_i8
    g = np.random.default_rng(3)
    dims, C = (12, 10, 8), 16
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, C)) for I in dims]
    U[1][3, 5] = np.nan  # q0 = mode 1 for n = 0
    U[0][2, 7] = np.inf  # q0 = mode 0 for n = 1, 2
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, 128 - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    M0 = mttkrp_i8(Td, dims, 0, Ud, C).cpu().numpy()
    assert np.all(np.isnan(M0[:, 5])) and np.all(np.isfinite(np.delete(M0, 5, axis=1)))
    M1 = mttkrp_i8(Td, dims, 1, Ud, C).cpu().numpy()
    assert np.all(np.isnan(M1[:, 7]))


@pytest.mark.parametrize("name,ps", [("tiny", range(10)), ("syn50_r3", range(50)), ("4way", [0, 1, 50, 99]),
                                     ("eem_r5", [0, 133, 267])])
def test_experimental_int8_sliced_fp64_path(name, ps):
    # precision JKCALS_FP64_I8: the whole JK-CALS loop with the INT8-sliced MTTKRP
    # held to the FP64 bar (1e-10) against the oracle
    from paper_2112_03985_b200 import JKCals
    w = make_workload(name)
    h = JKCals(w.T, w.R, hist_cap=w.sweeps, precision=2)
    h.set_init(w.P)
    h.iterate(w.sweeps, 0.0)
    ps = list(ps)
    res = O.jk_als(w.T, w.P, p_list=ps, max_iters=w.sweeps, nthreads=NCPU)
    check_against_oracle(h, res, ps, nt2p_of(w.T))


_RESIDENT_CHECK = r"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2112_03985_b200.jkcals import mttkrp_i8
worst = 0.0
for dims, C in [((37, 23, 11), 129), ((60, 50, 200), 250), ((13, 7, 5, 3), 70)]:
    g = np.random.default_rng(sum(dims) + C)
    T = np.asfortranarray(g.standard_normal(dims))
    U = [g.standard_normal((I, C)) for I in dims]
    ldu = ((C + 127) // 128) * 128
    Ud = [torch.from_numpy(np.pad(u, ((0, 0), (0, ldu - C)))).cuda() for u in U]
    Td = torch.from_numpy(np.ravel(T, order="F").copy()).cuda()
    for n in range(len(dims)):
        ref = O.mttkrp(T, U, n)
        M = mttkrp_i8(Td, dims, n, Ud, C).cpu().numpy()
        worst = max(worst, float(np.linalg.norm(M - ref) / np.linalg.norm(ref)))
print(worst)
"""


@pytest.mark.parametrize("env", [{"JKCALS_I8_RESIDENT": "1"}, {"JKCALS_I8_CLUSTER": "0"}])
def test_int8_kernel_variants(env):
    # the opt-in INT8 kernel variants -- resident A (JKCALS_I8_RESIDENT=1) and the one-CTA streaming
    # kernel (JKCALS_I8_CLUSTER=0); the knobs are read once per process, so each runs in a
    # subprocess -- meet the same bar as the default 2-CTA cluster kernel
    import subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _RESIDENT_CHECK], cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, **env), timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-13, out.stdout
