"""Critical path of a traced persistent-kernel launch: plan dump (H2B_DUMP_PLAN) + trace (.npy).
usage: critical_path.py plan.txt trace.npy"""
import sys
import numpy as np
plan = {}
for line in open(sys.argv[1]):
    if line.startswith("#"):
        print(line.strip()); continue
    a, b = line.split(":")
    q, ty, arg, cta, dur, fin, nlev = a.split()
    plan[int(q)] = dict(type=int(ty), arg=int(arg), cta=int(cta), dur=float(dur), nlev=int(nlev),
                        deps=[int(x) for x in b.split()])
t = np.load(sys.argv[2])
typ, arg, c, r, s, l0, l1, cd, d, sm = t.T.astype(np.float64)
t0 = c[c > 0].min()
us = lambda v: (v - t0) / 1e3
names = {0: "near", 1: "span", 2: "couple", 3: "flatup", 4: "flatdn"}
# walk back from the latest-finishing task through the dependency that finished last
cur = int(np.nanargmax(np.where(d > 0, d, np.nan)))
chain = []
while True:
    chain.append(cur)
    deps = [x for x in plan[cur]["deps"] if d[x] > 0]
    if not deps:
        break
    cur = max(deps, key=lambda x: d[x])
print("critical chain (latest-finishing dependency first-to-last):")
print(" qid  type   nlev   claim  ready  staged  computed  done   | wait-after-dep  staging  compute  out+flag")
prev_done = None
for q in reversed(chain):
    p = plan[q]
    gap = us(r[q]) - prev_done if prev_done is not None else float("nan")
    print(f"{q:5d} {names[p['type']]:6s} {p['nlev']:4d} {us(c[q]):7.2f} {us(r[q]):7.2f} {us(s[q]):7.2f} {us(cd[q]):8.2f} {us(d[q]):7.2f}"
          f"   | {gap:6.2f} {us(s[q]) - us(r[q]):7.2f} {us(cd[q]) - us(s[q]):7.2f} {us(d[q]) - us(cd[q]):7.2f}")
    prev_done = us(d[q])
