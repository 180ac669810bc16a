"""bench.py — JK-CALS on B200: seconds to fit all I_1 leave-one-out submodels (fixed sweeps).

Workload (BASELINE.json configs[3]): synthetic 200x200x200 tensor, planted rank 5,
1 % noise; rank-5 model; all 200 LOO submodels; 100 forced ALS sweeps;
FP64. One "step" = one full jackknife of this rank's shard: set_init (warm
start) + 100 sweeps of the fused MTTKRP + per-submodel epilogue + the jackknife moments of
modes 1..N-1 (all-gathered and Chan-merged across ranks), inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config NAME]
  torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU, NCCL)

Submodels are sharded contiguously over ranks (dist.shard); there is no per-iteration
communication. value = max over ranks of the device time (CUDA events) per step, in seconds
(strong scaling: the 200 submodels are fixed). The L2 (126 MB) is flushed between timed steps
because T (64 MB) fits in it. Roofline denominators: MEASURED_PEAKS.json (driver-written) for
HBM and bf16 (TF32 = bf16 x the guide's nominal 1.1/2.25); FP64 has no driver figure, so the
stricter of the builder-measured DMMA pipe peak (profiles/r01_fp64_microbench.txt) and a cuBLAS
DGEMM timed live here is used, labelled as such.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "jackknife s to fit all I1 submodels (fixed iters); MTTKRP TFLOP/s vs peak"
# FP64 DMMA.8x8x4 pipe peak measured by the builder on this pool (tools/microbench_fp64.cu,
# profiles/r01_fp64_microbench.txt): 148 SM x 128 FLOP/clk x 1.965 GHz
FP64_DMMA_PIPE_TFLOPS = 37.05
# INT8 tcgen05 (kind::i8) rate measured by the builder (profiles/r01_i8_microbench.txt): 8190
# MAC/clk/SM at N >= 128; the nominal dense figure is 4500 TOPS -- the stricter (larger) is used
I8_MEASURED_TOPS, I8_NOMINAL_TOPS = 4760.0, 4500.0


def measured_peaks():
    """MEASURED_PEAKS.json (driver-written), else the profiling guide's stated fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out = self.proc.communicate(timeout=5)[0]
            except Exception:
                out = ""
            self.lines = [l for l in out.strip().splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ oracle (CPU) legs
def cpu_baseline(w, sweeps_full, n_sub_full, sample_subs, sample_sweeps, threads):
    """Oracle JK-ALS (as it stands) on a bounded sample, extrapolated to the full job."""
    from oracle import oracle as O
    ps = list(np.linspace(0, w.dims[0] - 1, sample_subs).astype(int))
    t0 = time.perf_counter()
    O.jk_als(w.T, w.P, p_list=ps, max_iters=sample_sweeps, nthreads=threads)
    dt = time.perf_counter() - t0
    est = dt * (n_sub_full / len(ps)) * (sweeps_full / sample_sweeps)
    return est, dt, ps


def single_thread_baselines():
    """single-thread oracle timings of the small configs (full job; syn50 from a
    2-submodel sample extrapolated x25)."""
    from synth import make_workload
    out = {}
    for name, nsub in (("tiny", None), ("syn50_r5", 2)):
        w = make_workload(name)
        ns = nsub or w.dims[0]
        est, dt, _ = cpu_baseline(w, w.sweeps, w.dims[0], ns, w.sweeps, 1)
        out[name] = {"value": round(est, 4), "unit": "s", "threads": 1,
                     "sample": f"{ns} of {w.dims[0]} submodels x {w.sweeps} sweeps ({dt:.2f} s)"}
    return out


def run_reference(args):
    rank, _, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    from synth import make_workload
    w = make_workload(args.config)
    threads = os.cpu_count() or 1
    ss = min(threads, w.dims[0])
    vals = []
    for i in range(args.warmup + args.steps):
        est, dt, ps = cpu_baseline(w, w.sweeps, w.dims[0], ss, args.ref_sweeps, threads)
        if i >= args.warmup:
            vals.append(est)
    v = float(np.median(vals))
    sample = (f"oracle JK-ALS (plain C, {threads} threads over submodels) on {ss} of {w.dims[0]} submodels x "
              f"{args.ref_sweeps} of {w.sweeps} sweeps per step, extrapolated x{w.dims[0] / ss:.2f} x"
              f"{w.sweeps / args.ref_sweeps:.1f} to the full job")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(w, args),
            "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": threads, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def config_dict(w, args):
    return {"workload": f"{args.config}: synthetic {'x'.join(map(str, w.dims))}, rank {w.R}, all {w.dims[0]} "
                        f"LOO submodels, {w.sweeps} fixed ALS sweeps",
            "dims": list(w.dims), "rank": w.R, "n_submodels": w.dims[0], "sweeps": w.sweeps,
            "parallelism": f"submodel shards x{args.gpus}", "l2_flush": "256 MiB write between timed steps"}


# ------------------------------------------------------------------------------ GPU measurements
def live_dgemm_tflops(torch):
    """cuBLAS DGEMM 8192^3, best of 5 (a live FP64 denominator; cuBLAS is only the yardstick)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        best = ms if best is None else min(best, ms)
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def time_job(torch, h, init, sweeps, flush, reps, barrier=None):
    """Mean device time (CUDA events on the handle's stream) of set_init + `sweeps` fixed sweeps,
    after one untimed run; the L2 is flushed before each timed rep."""
    h.set_init(init)
    h.iterate(sweeps, 0.0)
    tot = 0.0
    for _ in range(reps):
        flush.random_(0, 255)
        (barrier or torch.cuda.synchronize)()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(h.stream)
        h.set_init(init)
        h.iterate(sweeps, 0.0)
        e.record(h.stream)
        e.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps / 1e3


def mttkrp_rate(h, init, sweeps, C, dims):
    """Instrumented (eager) pass: average MTTKRP launch time (CUDA events on the handle's stream)
    -> achieved TFLOP/s of the algorithmic 2 C prod(I) per launch."""
    h.set_init(init)
    h.set_instrument(True)
    h.iterate(sweeps, 0.0)
    t_m, t_e, nl = h.kernel_times()
    h.set_instrument(False)
    flops = 2.0 * C * float(np.prod(dims))
    avg_ms = float(t_m.sum()) / nl
    share = float(t_m.sum()) / float(t_m.sum() + t_e.sum())
    return flops / (avg_ms * 1e-3) / 1e12, avg_ms, flops, share


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="syn200")
    ap.add_argument("--ref-sweeps", type=int, default=30, help="sweeps per oracle sample step (~10 s on 16 cores)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: CPU collectives (N ranks may share one GPU: the path runs, timings are not scaling)")
    ap.add_argument("--dump-moments", default=None, help="rank 0 writes the merged jackknife moments here (.npz)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the supplementary FP32-path measurements")
    ap.add_argument("--no-i8", action="store_true", help="skip the supplementary FP64_I8-path measurement")
    ap.add_argument("--no-supp", action="store_true", help="skip the supplementary pool / delete-d / config lines")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2112_03985_b200 import JKCals
    from paper_2112_03985_b200.dist import allgather_moments, shard
    from paper_2112_03985_b200.jkcals import FP32, FP64_I8
    from synth import make_workload

    rank, local, world = dist_env()
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    coll_dev = torch.device("cuda", dev) if (world > 1 and args.dist_backend == "nccl") else torch.device("cpu")
    peaks = measured_peaks()
    w = make_workload(args.config)
    sb, se = shard(w.dims[0], world, rank)
    Td = torch.from_numpy(np.ravel(w.T, order="F").copy()).cuda()  # resident in HBM before timing
    h = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims)
    stream = h.stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    merged = {}

    def step():
        # one whole job: warm start, fixed sweeps, then the jackknife statistics of modes 1..N-1
        # (per-shard moments, all-gathered and Chan-merged when N > 1)
        h.set_init(w.P)
        h.iterate(w.sweeps, 0.0)
        for m in range(1, len(w.dims)):
            mom = h.local_moments(m)
            merged[m] = allgather_moments(mom) if world > 1 else mom

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x, op=None):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=op or dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()
    total_ms = 0.0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)  # L2 flush (outside the timed events)
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            step()
            e.record(stream)
            e.synchronize()
            total_ms += s.elapsed_time(e)
            barrier()
    ms = max_over_ranks(total_ms / args.steps)
    if args.dump_moments and rank == 0:
        np.savez(args.dump_moments, **{f"{k}_{m}": v for m, mom in merged.items()
                                       for k, v in zip(("count", "mean", "m2"), mom)})

    # --- roofline of the dominant kernel (fused MTTKRP), measured live with CUDA events on the
    # handle's stream in an instrumented (eager-launch) pass of one full job
    C_local = (se - sb) * w.R
    achieved, avg_launch_ms, flops_launch, mttkrp_share = mttkrp_rate(h, w.P, w.sweeps, C_local, w.dims)
    achieved = max_over_ranks(achieved, dist.ReduceOp.MIN if world > 1 else None)
    dgemm = live_dgemm_tflops(torch) if rank == 0 else None
    fp64_peak = max(FP64_DMMA_PIPE_TFLOPS, dgemm or 0.0)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r02_mttkrp_ncu_summary.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # --- end to end through the public API with HOST buffers (pinned, as a serving client would
    # hold them): H2D of T and P, create, set_init, 100 sweeps, D2H of every submodel's factors
    # + jackknife moments. One untimed run first (allocator / graph warm-up), then the median.
    T_pin = torch.empty(w.T.size, dtype=torch.float64, pin_memory=True)
    T_pin.numpy()[:] = np.ravel(w.T, order="F")
    P_pin = []
    for p in w.P:
        t_ = torch.empty(p.size, dtype=torch.float64, pin_memory=True)
        t_.numpy()[:] = np.ravel(p, order="F")
        P_pin.append((t_, t_.numpy().reshape(p.shape, order="F")))
    e2e_vals = []
    h2d = w.T.nbytes + sum(p.nbytes for p in w.P)
    d2h = 0
    for i in range(1 + max(3, min(args.steps, 5))):
        barrier()
        t0 = time.perf_counter()
        hh = JKCals(T_pin.numpy(), w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims)
        hh.set_init([pp[1] for pp in P_pin])
        hh.iterate(w.sweeps, 0.0)
        out = 0
        for m in range(len(w.dims)):  # every submodel's factors, one batched D2H per mode
            U_all, lam = hh.all_factors(m)
            out += U_all.nbytes + (lam.nbytes if m == len(w.dims) - 1 else 0)
        for m in range(1, len(w.dims)):
            mom = hh.local_moments(m)
            out += sum(x.nbytes for x in mom)
            if world > 1:
                allgather_moments(mom)
        torch.cuda.synchronize()
        if i > 0:
            e2e_vals.append(time.perf_counter() - t0)
        d2h = out
        hh.close()
    e2e = max_over_ranks(float(np.median(e2e_vals)))

    # set_init: N init_blocks + N gram + 1 reset; the sweeps; N - 1 moments kernels
    launches_per_step = (2 * len(w.dims) + 1) + h.launches_per_sweep() * w.sweeps + (len(w.dims) - 1)

    # --- supplementary: the FP64-accurate INT8-sliced path, same workload
    i8path = None
    if not args.no_i8:
        h8 = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims, precision=FP64_I8)
        t8 = time_job(torch, h8, w.P, w.sweeps, flush, max(2, min(args.steps, 3)), barrier)
        h8.set_init(w.P)
        h8.set_instrument(True)
        h8.iterate(w.sweeps, 0.0)
        tm8, _, nl8 = h8.kernel_times()
        ms8 = float(tm8.sum()) / nl8  # digits of U_q0 + the INT8 MMA kernel, per mode
        # the method's own digit products (unpadded): 28 of the 7 x 7 digit pairs, each a C x I_n x
        # I_q0 x J' contraction (2 ops per MAC); averaged over the N modes like the launches
        dd = list(w.dims)
        ops = 0.0
        for m in range(len(dd)):
            q0 = 1 if m == 0 else 0
            jp = float(np.prod([dd[k] for k in range(len(dd)) if k not in (m, q0)]))
            ops += 28 * 2 * C_local * dd[m] * dd[q0] * jp
        ops /= len(dd)
        tops = ops / (ms8 * 1e-3) / 1e12
        i8peak = max(I8_MEASURED_TOPS, I8_NOMINAL_TOPS)
        i8path = {"value": round(t8, 5), "unit": "s",
                  "dtype": "f64 results from int8 tcgen05 MMAs (7-digit operand slices, exact int32 accumulation)",
                  "mttkrp_fp64_equiv_tflops": round(flops_launch / (ms8 * 1e-3) / 1e12, 2),
                  "roofline": {"bound": "tensor", "unit": "TOPS (int8 MMA)", "achieved": round(tops, 1),
                               "peak": i8peak, "frac": round(tops / i8peak, 4),
                               "work": "unpadded digit products: 28 x 2 C I_n I_q0 J' per launch",
                               "peak_source": "builder-measured kind::i8 UMMA rate 8190 MAC/clk/SM at N >= 128 "
                                              "(profiles/r01_i8_microbench.txt; nominal dense 4500)"},
                  "status": "experimental (DESIGN.md §9b)"}
        h8.close()

    # --- supplementary: the optional FP32 path (3xTF32 on tcgen05, FP64 epilogue), same workload
    tf32_peak = round(peaks["bf16_tflops"] * 1.1 / 2.25, 1)
    fp32 = None
    if not args.no_fp32:
        h32 = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims, precision=FP32)
        t32 = time_job(torch, h32, w.P, w.sweeps, flush, max(2, min(args.steps, 3)), barrier)
        ach32, _, _, _ = mttkrp_rate(h32, w.P, w.sweeps, C_local, w.dims)
        fp32 = {"value": round(t32, 5), "unit": "s", "dtype": "f32 (3xTF32 tcgen05 MTTKRP, f64 epilogue)",
                "mttkrp_tflops_fp32_equiv": round(ach32, 2),
                "roofline": {"bound": "tensor", "achieved": round(3 * ach32, 2), "unit": "TFLOP/s (tf32 MMA)",
                             "peak": tf32_peak, "frac": round(3 * ach32 / tf32_peak, 4),
                             "peak_source": f"{peaks['source']} bf16 {peaks['bf16_tflops']} TF/s x nominal "
                                            "tf32/bf16 1.1/2.25"},
                "parity_bar": "1e-4 relative Frobenius vs the FP64 oracle"}
        h32.close()

    # --- supplementary (N = 1 only): the other named configs (north_star: throughput on the
    # synthetic and fluorescence-shaped workloads, absolute and vs roofline), the paper's "All"
    # pool (50 x 200 x 200, R in {3,5,7,9}) and delete-d, 100 fixed sweeps each
    supp, configs = None, None
    if world == 1 and not args.no_supp:
        from synth import make_pool
        configs = {}
        for name, prec in (("eem_r6", 0), ("4way", 0), ("4way", FP32)):
            wc = make_workload(name)
            hc = JKCals(wc.T, wc.R, hist_cap=wc.sweeps, precision=prec)
            tc = time_job(torch, hc, wc.P, wc.sweeps, flush, 2)
            Cc = wc.R * wc.dims[0]
            rate, avg_c, _, share_c = mttkrp_rate(hc, wc.P, wc.sweeps, Cc, wc.dims)
            key = name + ("_fp32" if prec == FP32 else "")
            if prec == FP32:
                roof = {"bound": "tensor", "achieved": round(3 * rate, 2), "unit": "TFLOP/s (tf32 MMA)",
                        "peak": tf32_peak, "frac": round(3 * rate / tf32_peak, 4)}
            else:
                roof = {"bound": "tensor", "achieved": round(rate, 3), "unit": "TFLOP/s", "peak": fp64_peak,
                        "frac": round(rate / fp64_peak, 4)}
            configs[key] = {"workload": f"{name}: {'x'.join(map(str, wc.dims))}, rank {wc.R}, all {wc.dims[0]} LOO "
                                        f"submodels, {wc.sweeps} fixed sweeps, {'FP32 path' if prec else 'FP64'}",
                            "value": round(tc, 5), "unit": "s", "mttkrp_tflops": round(rate, 2),
                            "avg_launch_ms": round(avg_c, 4), "share_of_step": round(share_c, 4), "roofline": roof}
            hc.close()
        pw = make_pool("all_medium")
        hp = JKCals(pw.T, list(pw.ranks), hist_cap=pw.sweeps)
        tp = time_job(torch, hp, pw.Ps, pw.sweeps, flush, 2)
        fl_p = hp.sweep_flops() * pw.sweeps
        hp.close()
        dd = 10
        hd = JKCals(Td, w.R, hist_cap=w.sweeps, dims=w.dims, d=dd)
        td = time_job(torch, hd, w.P, w.sweeps, flush, 2)
        fl_d = hd.sweep_flops() * w.sweeps
        hd.close()
        # small configs (SURVEY §8d latency targets): whole-iterate time per sweep, auto path
        # (warp-resident kernel for tiny, cluster-resident for syn50 R1-R2, streamed otherwise)
        lat = {}
        for name in ("tiny", "syn50_r1", "syn50_r2", "syn50_r3", "syn50_r5"):
            wl = make_workload(name)
            nsw = 1000 if name == "tiny" else 200
            hl = JKCals(wl.T, wl.R, hist_cap=nsw)
            tl = time_job(torch, hl, wl.P, nsw, flush, 3)
            lat[name] = round(tl / nsw * 1e6, 2)
            hl.close()
        supp = {
            "latency_us_per_sweep": lat,
            "all_pool": {"workload": "all_medium: 50x200x200, models R in {3,5,7,9} jackknifed together "
                                     "(200 submodels, C = 1200), 100 sweeps", "value": round(tp, 5), "unit": "s",
                         "mttkrp_flop_rate_tflops": round(fl_p / tp / 1e12, 2)},
            "delete_d": {"workload": f"{args.config} delete-{dd} jackknife ({-(-w.dims[0] // dd)} groups), "
                                     f"{w.sweeps} sweeps", "value": round(td, 5), "unit": "s",
                         "mttkrp_flop_rate_tflops": round(fl_d / td / 1e12, 2)},
        }

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            ss = min(threads, w.dims[0])
            est, dt, ps = cpu_baseline(w, w.sweeps, w.dims[0], ss, args.ref_sweeps, threads)
            cpu = {"value": round(est, 2), "unit": "s", "cores": threads, "kind": "oracle",
                   "sample": f"oracle JK-ALS on {ss} of {w.dims[0]} submodels x {args.ref_sweeps} of "
                             f"{w.sweeps} sweeps ({dt:.1f} s on {threads} threads), extrapolated to the full job",
                   "cpu_model": cpu_model(), "single_thread": single_thread_baselines()}
        csum = clk.summary()
        line = {
            "metric": METRIC, "value": round(ms / 1e3, 5), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded planted CP tensor + noise)",
            "config": dict(config_dict(w, args), dist_backend=args.dist_backend if world > 1 else None),
            "mttkrp_tflops": round(achieved, 2),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": round(achieved / fp64_peak, 4), "traffic": traffic,
                         "kernel": "mttkrp_dmma_kernel (FP64 DMMA)", "flops_per_launch": flops_launch,
                         "avg_launch_ms": round(avg_launch_ms, 4), "share_of_step": round(mttkrp_share, 4),
                         "frac_of_live_cublas_dgemm": round(achieved / dgemm, 4) if dgemm else None,
                         # the JK-ALS-useful share of the padded work, (I_0 - 1) / I_0
                         "useful_tflops": round(achieved * (w.dims[0] - 1) / w.dims[0], 3),
                         "peak_source": f"max(builder-measured DMMA pipe {FP64_DMMA_PIPE_TFLOPS} TF/s "
                                        f"(profiles/r01_fp64_microbench.txt), cuBLAS DGEMM 8192^3 timed live "
                                        f"{round(dgemm, 2) if dgemm else None} TF/s); MEASURED_PEAKS.json has no FP64 entry"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e, 4), "unit": "s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches_per_step * args.steps),
            "fp32_path": fp32,
            "fp64_int8_path": i8path,
            "configs": configs,
            "supplementary": supp,
            "peaks": peaks,
            "clocks": {"sm_mhz": csum["sm_mhz"], "sm_max_mhz": csum["sm_max_mhz"], "reasons": csum["reasons"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
