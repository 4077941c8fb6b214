"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.
    python profiles/launch_summary.py gpurun_out/launches_r01.csv"""
import csv
import io
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
agg = defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    agg[k][0] += 1
    agg[k][1] += float(r["Metric Value"]) * scale[r["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {v[0]:8d} {v[1]:10.2f} {1e3 * v[1] / v[0]:9.1f} {100 * v[1] / tot:5.1f}%")
