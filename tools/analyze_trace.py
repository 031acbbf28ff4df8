"""Summarise a persistent-kernel trace (tools/trace_mega.py output, 8 columns per task)."""
import sys
import numpy as np
t = np.load(sys.argv[1])
typ, arg, c, r, s, l0, l1, cd, d, sm = t.T
t0 = c[c > 0].min()
f = lambda v: np.where(v > 0, (v - t0) / 1e3, np.nan)
c, r, s, l0, l1, cd, d = f(c), f(r), f(s), f(l0), f(l1), f(cd), f(d)
names = {0: "near", 1: "span", 2: "couple", 3: "flatup", 4: "flatdn"}
print(f"makespan {np.nanmax(d):.1f} us, tasks {len(t)}, CTAs {len(np.unique(sm >> 32))}")
for ty in (0, 1, 2):
    m = typ == ty
    if not m.any():
        continue
    wait, run = r[m] - c[m], d[m] - r[m]
    extra = ""
    if ty == 1:
        extra = (f" | staging {np.nanmean(s[m] - r[m]):5.2f} lvl0 {np.nanmean(l0[m] - s[m]):5.2f} "
                 f"lvl1 {np.nanmean(l1[m] - l0[m]):5.2f} compute {np.nanmean(cd[m] - s[m]):5.2f} "
                 f"stage-out+flag {np.nanmean(d[m] - cd[m]):5.2f}")
    print(f"{names[ty]:7s} n={m.sum():5d} claim[{np.nanmin(c[m]):6.1f},{np.nanmax(c[m]):6.1f}] done_max={np.nanmax(d[m]):6.1f} "
          f"wait mean={np.nanmean(wait):6.2f} max={np.nanmax(wait):6.2f} run mean={np.nanmean(run):6.2f} max={np.nanmax(run):6.2f}{extra}")
# critical chain: walk back from the last task through the latest-finishing dependency is not
# recorded; show far tasks sorted by ready time
idx = np.nonzero(typ != 0)[0]
order = idx[np.argsort(r[idx])]
print("far tasks by ready time (id type ready staged computed done):")
step = max(1, len(order) // 14)
for i in list(order[::step]) + [order[-1]]:
    print(f"  {i:5d} {names[typ[i]]:6s} {r[i]:7.2f} {s[i]:7.2f} {cd[i]:7.2f} {d[i]:7.2f}")
T = np.nanmax(d)
nb = 20
bins = np.linspace(0, T, nb + 1)
busy = np.zeros(nb)
for ci, di in zip(r, d):
    for b in range(nb):
        busy[b] += max(0.0, min(bins[b + 1], di) - max(bins[b], ci))
ncta = len(np.unique(sm >> 32))
print("busy fraction per 5%:", " ".join(f"{x / ((bins[1] - bins[0]) * ncta):.2f}" for x in busy))
