"""Walk the SASS page of an ncu report: stall samples accumulated between
synchronisation / memory instructions (where a persistent kernel spends its time).

python tools/ncu_walk.py report.ncu-rep [min_pct]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = rows[2:]
idx = {k: i for i, k in enumerate(h)}
stalls = ["stall_barrier", "stall_lg", "stall_long_sb", "stall_math", "stall_mio", "stall_short_sb", "stall_wait",
          "stall_not_selected", "stall_dispatch"]


def S(r, k):
    v = r[idx[k]]
    return int(v) if v else 0


tot = sum(S(r, "# Samples") for r in data)
print(rows[0][1][:120], "samples", tot)
win = dict.fromkeys(stalls, 0)
acc = 0
for i, r in enumerate(data):
    s = S(r, "# Samples")
    src = r[idx["Source"]]
    if any(m in src for m in ("BAR.", "SYNCS.PHASECHK", "SYNCS.ARRIVE", "USETMAXREG", "EXIT", "LDG", "STG")):
        if acc > thr / 100 * tot:
            print(f"{i:5d} win={acc/tot*100:5.1f}% ",
                  {k[6:]: round(v / tot * 100, 1) for k, v in win.items() if v > 0.003 * tot}, "|", src[:60],
                  f" self={s/tot*100:.1f}%")
        acc = 0
        win = dict.fromkeys(stalls, 0)
    acc += s
    for k in stalls:
        win[k] += S(r, k)
