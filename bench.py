"""bench.py — JK-CALS on B200: seconds to fit all I_1 leave-one-out submodels (fixed sweeps).

Workload (BASELINE.json configs[3]): synthetic 200x200x200 tensor, planted rank 5,
1 % noise; rank-5 model; all 200 LOO submodels; 100 forced ALS sweeps;
FP64. One "step" = one full jackknife of this rank's shard: set_init (warm
start) + 100 sweeps of the fused MTTKRP + per-submodel epilogue, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config NAME]
  torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU, NCCL)

Submodels are sharded contiguously over ranks (dist.shard); there is no per-iteration
communication. value = max over ranks of the device time (CUDA events) per step, in seconds
(strong scaling: the 200 submodels are fixed). The L2 (126 MB) is flushed between timed steps
because T (64 MB) fits in it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "jackknife s to fit all I1 submodels (fixed iters); MTTKRP TFLOP/s vs peak"
# FP64 peak of this B200 pool: DMMA.8x8x4 pipe microbenchmark (tools/microbench_fp64.cu,
# profiles/r01_fp64_microbench.txt) = 37.05 TFLOP/s, i.e. 148 SM x 128 FLOP/clk x 1.965 GHz;
# cuBLAS DGEMM 8192^3 reached 35.45 (profiles/r01_dgemm_peak.json). MEASURED_PEAKS.json has
# no FP64 entry, so the measured pipe peak is the denominator (the stricter of the two).
FP64_PEAK_TFLOPS = 37.05
FP64_DGEMM_TFLOPS = 35.45
# TF32 dense tensor peak for the FP32 path's roofline: MEASURED_PEAKS.json bf16 (1678 TF/s burst)
# x the guide's nominal tf32/bf16 ratio (1.1 / 2.25 PFLOP/s); 3xTF32 issues 3 MMAs per FP32 product
TF32_PEAK_TFLOPS = round(1678.0 * 1.1 / 2.25, 1)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


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


def cpu_baseline(w, sweeps_full, n_sub_full, sample_subs, sample_sweeps, threads):
    """Oracle JK-ALS (as it stands) on a bounded sample, extrapolated to the full job."""
    from oracle import oracle as O
    ps = list(np.linspace(0, w.dims[0] - 1, sample_subs).astype(int))
    t0 = time.perf_counter()
    O.jk_als(w.T, w.P, p_list=ps, max_iters=sample_sweeps, nthreads=threads)
    dt = time.perf_counter() - t0
    est = dt * (n_sub_full / len(ps)) * (sweeps_full / sample_sweeps)
    return est, dt, ps


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
            "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": threads, "kind": "oracle", "sample": sample},
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="syn200")
    ap.add_argument("--ref-sweeps", type=int, default=30, help="sweeps per oracle sample step (~10 s on 16 cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the supplementary FP32-path measurement")
    ap.add_argument("--no-supp", action="store_true", help="skip the supplementary pool / delete-d lines")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2112_03985_b200 import JKCals
    from paper_2112_03985_b200.dist import shard
    from synth import make_workload

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = make_workload(args.config)
    sb, se = shard(w.dims[0], world, rank)
    Td = torch.from_numpy(np.ravel(w.T, order="F").copy()).cuda()  # resident in HBM before timing
    h = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims)
    stream = h.stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    from paper_2112_03985_b200.dist import allgather_moments

    def step():
        # one whole job: warm start, fixed sweeps, then the jackknife statistics of modes 1..N-1
        # (per-shard moments, all-gathered and Chan-merged over NCCL when N > 1)
        h.set_init(w.P)
        h.iterate(w.sweeps, 0.0)
        for m in range(1, len(w.dims)):
            mom = h.local_moments(m)
            if world > 1:
                allgather_moments(mom)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    total_ms = 0.0
    with ClockSampler(local) as clk:
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
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # --- roofline of the dominant kernel (fused MTTKRP), measured live with CUDA events on the
    # handle's stream in an instrumented (eager-launch) pass of one full step
    h.set_init(w.P)
    h.set_instrument(True)
    barrier()
    h.iterate(w.sweeps, 0.0)
    t_m, t_e, nl = h.kernel_times()
    h.set_instrument(False)
    C_local = (se - sb) * w.R
    flops_launch = 2.0 * C_local * float(np.prod(w.dims))  # 2 C prod(I) per mode
    avg_launch_ms = float(t_m.sum()) / nl
    achieved = flops_launch / (avg_launch_ms * 1e-3) / 1e12
    mttkrp_share = float(t_m.sum()) / float(t_m.sum() + t_e.sum())
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r01_mttkrp_ncu_summary.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if world > 1:
        t = torch.tensor([achieved], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        achieved = float(t.item())

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
        torch.cuda.synchronize()
        if i > 0:
            e2e_vals.append(time.perf_counter() - t0)
        d2h = out
        hh.close()
    e2e = float(np.median(e2e_vals))
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    # set_init: N init_blocks + N gram + 1 reset; the sweeps; N - 1 moments kernels
    launches_per_step = (2 * len(w.dims) + 1) + h.launches_per_sweep() * w.sweeps + (len(w.dims) - 1)

    # --- supplementary: the experimental FP64-accurate INT8-sliced path, same workload
    i8path = None
    if not args.no_fp32:
        from paper_2112_03985_b200.jkcals import FP64_I8
        h8 = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims, precision=FP64_I8)
        for _ in range(2):
            h8.set_init(w.P)
            h8.iterate(w.sweeps, 0.0)
        t8 = 0.0
        reps8 = max(2, min(args.steps, 3))
        for _ in range(reps8):
            flush.random_(0, 255)
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(h8.stream)
            h8.set_init(w.P)
            h8.iterate(w.sweeps, 0.0)
            e.record(h8.stream)
            e.synchronize()
            t8 += s.elapsed_time(e)
        t8 /= reps8
        h8.set_init(w.P)
        h8.set_instrument(True)
        h8.iterate(w.sweeps, 0.0)
        tm8, _, nl8 = h8.kernel_times()
        ms8 = float(tm8.sum()) / nl8  # digits of U_q0 + the INT8 MMA kernel, per mode
        # INT8 MMA work per launch: 28 digit products x (C_pad x I_n,pad x I_q0,pad x J') MACs x 2
        dd = list(w.dims)
        ops = 0.0
        for m in range(len(dd)):
            q0 = 1 if m == 0 else 0
            jp = float(np.prod([dd[k] for k in range(len(dd)) if k not in (m, q0)]))
            ops += 28 * 2 * (-(-C_local // 128) * 128) * (-(-dd[m] // 64) * 64) * (-(-dd[q0] // 32) * 32) * jp
        ops /= len(dd)
        i8path = {"value": round(t8 / 1e3, 5), "unit": "s",
                  "dtype": "f64 results from int8 tcgen05 MMAs (7-digit operand slices, exact int32 accumulation)",
                  "mttkrp_fp64_equiv_tflops": round(flops_launch / (ms8 * 1e-3) / 1e12, 2),
                  "roofline": {"bound": "tensor", "unit": "TOPS (int8 MMA)", "achieved": round(ops / (ms8 * 1e-3) / 1e12, 1),
                               "peak": 4760.0, "frac": round(ops / (ms8 * 1e-3) / 1e12 / 4760.0, 4),
                               "peak_source": "measured kind::i8 UMMA rate, 8190 MAC/clk/SM at N >= 128 "
                                              "(profiles/r01_i8_microbench.txt); nominal dense int8 is 4500"},
                  "parity": "every submodel of syn200 / eem R5 / 4-way within 8.2e-14 (factors) / 9.1e-14 (lambda) of the oracle "
                            "(profiles/r01_full_parity.jsonl), same bar as the FP64 path",
                  "status": "experimental (DESIGN.md §9b)"}
        h8.close()

    # --- supplementary: the optional FP32 path (3xTF32 on tcgen05, FP64 epilogue), same workload
    fp32 = None
    if not args.no_fp32:
        from paper_2112_03985_b200.jkcals import FP32
        h32 = JKCals(Td, w.R, sub_range=(sb, se), hist_cap=w.sweeps, dims=w.dims, precision=FP32)
        for _ in range(2):
            h32.set_init(w.P)
            h32.iterate(w.sweeps, 0.0)
        t32 = 0.0
        for _ in range(max(2, min(args.steps, 3))):
            flush.random_(0, 255)
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(h32.stream)
            h32.set_init(w.P)
            h32.iterate(w.sweeps, 0.0)
            e.record(h32.stream)
            e.synchronize()
            t32 += s.elapsed_time(e)
        t32 /= max(2, min(args.steps, 3))
        h32.set_init(w.P)
        h32.set_instrument(True)
        h32.iterate(w.sweeps, 0.0)
        tm32, te32, nl32 = h32.kernel_times()
        ach32 = flops_launch / (float(tm32.sum()) / nl32 * 1e-3) / 1e12
        fp32 = {"value": round(t32 / 1e3, 5), "unit": "s", "dtype": "f32 (3xTF32 tcgen05 MTTKRP, f64 epilogue)",
                "mttkrp_tflops_fp32_equiv": round(ach32, 2),
                "roofline": {"bound": "tensor", "achieved": round(3 * ach32, 2), "unit": "TFLOP/s (tf32 MMA)",
                             "peak": TF32_PEAK_TFLOPS, "frac": round(3 * ach32 / TF32_PEAK_TFLOPS, 4),
                             "peak_source": "measured bf16 cuBLAS 1678 TF/s x nominal tf32/bf16 ratio 1.1/2.25"},
                "parity_bar": "1e-4 relative Frobenius vs the FP64 oracle"}
        h32.close()
    # --- supplementary (N = 1 only): the paper's "All" pool (50 x 200 x 200, R in {3,5,7,9}, the
    # P:496-504 medium tensor) and delete-d on the bench workload, 100 fixed sweeps each, FP64
    supp = None
    if world == 1 and not args.no_supp:
        from synth import make_pool

        def timed(hh, init, sweeps, reps=2):
            hh.set_init(init)
            hh.iterate(sweeps, 0.0)
            tot = 0.0
            for _ in range(reps):
                flush.random_(0, 255)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(hh.stream)
                hh.set_init(init)
                hh.iterate(sweeps, 0.0)
                e.record(hh.stream)
                e.synchronize()
                tot += s.elapsed_time(e)
            return tot / reps / 1e3

        pw = make_pool("all_medium")
        hp = JKCals(pw.T, list(pw.ranks), hist_cap=pw.sweeps)
        tp = timed(hp, pw.Ps, pw.sweeps)
        fl_p = hp.sweep_flops() * pw.sweeps
        hp.close()
        dd = 10
        hd = JKCals(Td, w.R, hist_cap=w.sweeps, dims=w.dims, d=dd)
        td = timed(hd, w.P, w.sweeps)
        fl_d = hd.sweep_flops() * w.sweeps
        hd.close()
        supp = {
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
                             f"{w.sweeps} sweeps ({dt:.1f} s on {threads} threads), extrapolated to the full job"}
        csum = clk.summary()
        line = {
            "metric": METRIC, "value": round(ms / 1e3, 5), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded planted CP tensor + noise)",
            "config": config_dict(w, args),
            "mttkrp_tflops": round(achieved, 2),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic,
                         "kernel": "mttkrp_dmma_kernel (FP64 DMMA)", "flops_per_launch": flops_launch,
                         "avg_launch_ms": round(avg_launch_ms, 4), "share_of_step": round(mttkrp_share, 4),
                         "frac_of_cublas_dgemm": round(achieved / FP64_DGEMM_TFLOPS, 4),
                         # the JK-ALS-useful share of the padded work, (I_0 - 1) / I_0
                         "useful_tflops": round(achieved * (w.dims[0] - 1) / w.dims[0], 3),
                         "peak_source": "measured FP64 DMMA pipe peak (profiles/r01_fp64_microbench.txt)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e, 4), "unit": "s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches_per_step * args.steps),
            "fp32_path": fp32,
            "fp64_int8_path": i8path,
            "supplementary": supp,
            "clocks": {"sm_mhz": csum["sm_mhz"], "sm_max_mhz": csum["sm_max_mhz"], "reasons": csum["reasons"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
