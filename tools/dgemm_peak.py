"""Measure cuBLAS FP64 DGEMM throughput (burst best-of-10 and ~4 s sustained), the
roofline denominator for the FP64 MTTKRP ('the sustained FP64 DGEMM peak
measured on the box')."""
import json, subprocess, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = a @ b; torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); c = a @ b; e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
burst = 2 * n ** 3 / (best * 1e-3) / 1e12
clk = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cnt = 0; t0 = time.time(); s.record()
while time.time() - t0 < 4.0:
    for _ in range(4): c = a @ b
    cnt += 4
    torch.cuda.synchronize()
e.record(); e.synchronize()
sus = 2 * n ** 3 * cnt / (s.elapsed_time(e) * 1e-3) / 1e12
clk.terminate(); lines = clk.stdout.read().strip().splitlines()
print(json.dumps({"dgemm_fp64_tflops_burst": round(burst, 2), "dgemm_fp64_tflops_sustained": round(sus, 2),
                  "n": n, "clock_samples": lines[-8:]}))
