"""SURVEY §8(d) secondary, the paper's Fig. 1 analog: MTTKRP efficiency
against the fused width C on a 50 x 200 x 200 tensor. C = K x 8 columns of K rank-8 CALS models fused
into one MTTKRP (d = 0 pool); per-mode average launch time of the FP64 DMMA MTTKRP
from an instrumented pass (CUDA events), algorithmic 2 C prod(I) flops per launch, against the
37.05 TF/s DMMA peak. One JSON line per C."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2112_03985_b200 import cals

PEAK = 37.05
dims = (50, 200, 200)
rng = np.random.default_rng(0)
T = rng.standard_normal(dims)
P = float(np.prod(dims))
for C in (16, 32, 64, 128, 256, 512, 1024, 2048):
    R = 8
    K = C // R
    inits = [[rng.standard_normal((I, R)) for I in dims] for _ in range(K)]
    h = cals(T, [R] * K, inits, hist_cap=8)
    h.iterate(2, 0.0)
    h.set_init(inits)
    h.set_instrument(True)
    sweeps = 6
    h.iterate(sweeps, 0.0)
    tm, te, _ = h.kernel_times()  # ms, summed over the sweeps, per mode
    per_mode = [2.0 * C * P / (t / sweeps * 1e-3) / 1e12 for t in tm]
    avg_us = float(np.mean(tm)) / sweeps * 1e3
    rate = 2.0 * C * P / (avg_us * 1e-6) / 1e12
    print(json.dumps({"C": C, "models": K, "rank": R, "avg_launch_us": round(avg_us, 2),
                      "mttkrp_tflops": round(rate, 2), "frac_of_dmma_peak": round(rate / PEAK, 3),
                      "per_mode_tflops": [round(x, 2) for x in per_mode],
                      "epilogue_us_per_mode": [round(t / sweeps * 1e3, 2) for t in te]}), flush=True)
    h.close()
