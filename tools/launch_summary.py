"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv) over the
last N timed steps.  Usage: python tools/launch_summary.py gpurun_out/launches.csv [steps]"""
import csv, sys
from collections import OrderedDict

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
for r in rd:
    if r[mi] == "gpu__time_duration.sum":
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        rows.append((r[ki], float(r[vi].replace(",", "")) * scale))
# a step starts at the embedding gather
starts = [i for i, (k, _) in enumerate(rows) if "embed_kernel" in k]
first = starts[-steps] if len(starts) >= steps else 0
sel = rows[first:]
tot = OrderedDict()
for k, t in sel:
    name = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    c, s = tot.get(name, (0, 0.0))
    tot[name] = (c + 1, s + t)
all_us = sum(s for _, s in tot.values())
print(f"Last {steps} steps: {len(sel)} launches, {all_us / steps:.1f} us per step (sum of kernel durations)\n")
print("| kernel | launches/step | us/step | share |")
print("|---|---|---|---|")
for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {c // steps} | {s / steps:.0f} | {100 * s / all_us:.1f}% |")
