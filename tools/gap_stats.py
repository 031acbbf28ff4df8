"""Dependency-to-ready gaps of a traced persistent-kernel launch (plan dump + trace .npy).
usage: gap_stats.py plan.txt trace.npy"""
import sys
import numpy as np
plan = {}
for line in open(sys.argv[1]):
    if line.startswith("#"):
        continue
    a, b = line.split(":")
    qq, ty, arg, cta, dur, fin, nlev = a.split()
    plan[int(qq)] = dict(type=int(ty), deps=sorted(set(int(x) for x in b.split())))
t = np.load(sys.argv[2]).astype(np.float64)
c, r, d = t[:, 2], t[:, 3], t[:, 8]
names = {1: "span", 2: "couple", 3: "flatup", 4: "flatdn"}
rows = []
for q, p in plan.items():
    if not p["deps"]:
        continue
    md = max(d[x] for x in p["deps"])
    start = max(md, c[q])
    rows.append((p["type"], (r[q] - start) / 1e3, len(p["deps"]), c[q] > md))
rows = np.array(rows)
for ty in np.unique(rows[:, 0]):
    m = rows[:, 0] == ty
    g = rows[m, 1]
    print(f"{names[int(ty)]:7s} n={m.sum():4d} gap(ready - max(dep done, claim)) mean {g.mean():.2f} p50 {np.median(g):.2f} "
          f"p90 {np.percentile(g, 90):.2f} max {g.max():.2f} us; deps mean {rows[m, 2].mean():.1f}; "
          f"claimed after deps done {rows[m, 3].mean() * 100:.0f}%")
