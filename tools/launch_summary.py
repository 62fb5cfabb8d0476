"""Summarise an ncu launch list (gpu__time_duration.sum per launch): count, mean and share per kernel.

usage: python tools/launch_summary.py gpurun_out/launches.csv  (per-launch times are cold-cache
and serialised; compare shares, not absolutes)
"""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
lines = [l for l in text.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
    agg[r[ki]].append(v * scale)
step_kernels = [k for k in agg if "feas_level" not in k and "dfma" not in k]
tot = sum(sum(agg[k]) for k in step_kernels)
print("%-60s %6s %14s %14s" % ("kernel", "count", "mean_ns", "share_of_step"))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = "%.4f" % (sum(v) / tot) if k in step_kernels else "setup"
    print("%-60s %6d %14.0f %14s" % (k[:60], len(v), sum(v) / len(v), share))
