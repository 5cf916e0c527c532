"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
launches, total device time and share per kernel (cold-cache, serialised
times: compare shares, not absolutes).

python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/<name>_summary.txt
"""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
lines = [ln for ln in text.splitlines() if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
    k = r["Kernel Name"]
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of")
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}   (cold-cache, serialised: compare shares)")
print("launches   total_us  share  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{cnt[k]:8d} {v:10.1f} {v / s * 100:5.1f}%  {k[:110]}")
