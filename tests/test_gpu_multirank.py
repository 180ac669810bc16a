"""The N > 1 path of bench.py, executed: two ranks under torch.distributed.run on one B200.

Both ranks share the one GPU of the test box (gloo collectives; no kernel waits on another
rank, so this exercises the sharded path -- contiguous shards, replicated T, max-over-ranks
timing, the in-step all-gather + Chan merge of the jackknife moments and the N = 2 JSON line --
without pretending to measure scaling). The merged moments must equal those of one process
fitting all submodels (concurrent instances are independent).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo_on_one_gpu(tmp_path):
    from paper_2112_03985_b200 import JKCals
    from synth import make_workload

    dump = str(tmp_path / "moments.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--dist-backend", "gloo", "--no-cpu-baseline",
           "--no-fp32", "--no-i8", "--no-supp", "--dump-moments", dump]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 1 and line["warmup"] == 3
    assert line["metric"].startswith("jackknife s") and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"] == "submodel shards x2"
    assert line["roofline"]["achieved"] > 0 and line["gpu_launches"] > 0

    w = make_workload("syn200")
    h = JKCals(w.T, w.R, hist_cap=w.sweeps)
    h.set_init(w.P)
    h.iterate(w.sweeps, 0.0)
    got = np.load(dump)
    for m in (1, 2):
        c, mean, m2 = h.local_moments(m)
        assert np.array_equal(got[f"count_{m}"], c)
        assert np.allclose(got[f"mean_{m}"], mean, rtol=1e-13, atol=1e-15)
        assert np.allclose(got[f"m2_{m}"], m2, rtol=1e-9, atol=1e-12 * np.abs(m2).max())
