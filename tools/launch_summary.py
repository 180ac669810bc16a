"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launches,
total / average time and share (cold-cache, serialised: compare shares, not absolutes)."""
import csv, io, json, re, sys
from collections import OrderedDict

path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
lines = [l for l in open(path) if l.startswith('"')]
agg = OrderedDict()
for r in csv.DictReader(io.StringIO("".join(lines))):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r["Kernel Name"])
    name = re.sub(r"^void ", "", name).replace("jk::", "")
    v = float(r["Metric Value"]) / 1e3  # ns -> us
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
out = {"command": cmd, "note": "cold-cache serialised per-launch timings: compare shares, not absolutes",
       "kernels": [{"kernel": k, "launches": n, "total_us": round(t, 2), "avg_us": round(t / n, 3),
                    "share": round(t / tot, 4)} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}
print(json.dumps(out, indent=1))
