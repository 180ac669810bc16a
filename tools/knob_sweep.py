"""Dev: time one submodel shard under several tuning-knob settings (each in its own process, the
knobs being read once): knob_sweep.py <workload> <nsub> '<ENV=V ...>' ['<ENV=V ...>' ...]."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys
sys.path.insert(0, %r)
import torch
from paper_2112_03985_b200 import JKCals
from synth import make_workload
w = make_workload(sys.argv[1]); nsub = int(sys.argv[2])
h = JKCals(w.T, w.R, hist_cap=100, sub_range=(0, nsub))
best = 1e30
for rep in range(3):
    h.set_init(w.P)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(h.stream); h.iterate(100, 0.0); e.record(h.stream); e.synchronize()
    best = min(best, s.elapsed_time(e))
print(best)
""" % ROOT
wl, nsub = sys.argv[1], sys.argv[2]
for spec in sys.argv[3:] or [""]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD, wl, nsub], env=env, capture_output=True, text=True)
    ms = float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else None
    print(json.dumps({"workload": wl, "nsub": int(nsub), "knobs": spec, "ms_100_sweeps": ms,
                      "err": None if ms else out.stderr[-300:]}), flush=True)
