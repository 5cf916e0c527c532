"""Sweep ring configurations (NB, S) per (dtype, b) with B200WD_RING_CFG in
fresh processes; prints the best per case.
python tools/tune_ring.py [dtype:b ...] [--nbs 1,2,4] [--depths 2,3,4,6]"""
import itertools
import os
import re
import subprocess
import sys

args = sys.argv[1:]
opt = {k: [int(x) for x in args[i + 1].split(",")] for i, k in enumerate(args) if k in ("--nbs", "--depths")}
pos = [a for i, a in enumerate(args) if not a.startswith("--") and (i == 0 or args[i - 1] not in ("--nbs", "--depths"))]
cases = [(a.split(":")[0], int(a.split(":")[1])) for a in pos] or (
    [("c128", b) for b in (4, 6, 8, 12, 16, 24, 32)] + [("c64", b) for b in (4, 6, 8, 12, 16, 24, 32)])
cfgs = [(nb, s) for nb in opt.get("--nbs", (1, 2, 4)) for s in opt.get("--depths", (2, 3, 4, 6))]
best = {}
for dt, b in cases:
    res = []
    for nb, s in cfgs:
        env = dict(os.environ, B200WD_RING_CFG=f"{nb},{s}")
        out = subprocess.run([sys.executable, "tools/sweep_dirac.py", "--dtypes", dt, "--bs", str(b), "--iters", "30"],
                             env=env, capture_output=True, text=True).stdout
        m = re.search(r"([0-9.]+) ms .* frac ([0-9.]+)", out)
        if m:
            res.append((float(m.group(1)), nb, s, float(m.group(2))))
    res.sort()
    res.append((float("inf"), 0, 0, 0.0))
    env = dict(os.environ)
    env.pop("B200WD_RING_CFG", None)
    out = subprocess.run([sys.executable, "tools/sweep_dirac.py", "--dtypes", dt, "--bs", str(b), "--iters", "30"],
                         env=env, capture_output=True, text=True).stdout
    m = re.search(r"([0-9.]+) ms .* frac ([0-9.]+)", out)
    if m:
        res[-1] = (float(m.group(1)), 0, 0, float(m.group(2)))  # 0,0 = the shipped table/default
    res.sort()
    print(dt, b, " ".join(f"{nb},{s}:{f:.3f}" for t, nb, s, f in res[:5]), flush=True)
    best[(dt, b)] = res[0] if res else None
print("BEST", {f"{k[0]}_{k[1]}": (v[1], v[2], v[3]) for k, v in best.items() if v})
