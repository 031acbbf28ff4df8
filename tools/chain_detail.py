"""Critical chain of a traced launch with each task's CTA predecessors (plan dump + trace).
usage: chain_detail.py plan.txt trace.npy"""
import sys
import numpy as np
plan = {}
for line in open(sys.argv[1]):
    if line.startswith("#"):
        print(line.strip()); continue
    a, b = line.split(":")
    qq, ty, arg, cta, dur, fin, nlev = a.split()
    plan[int(qq)] = dict(type=int(ty), cta=int(cta), dur=float(dur), fin=float(fin), deps=[int(x) for x in b.split()])
t = np.load(sys.argv[2]).astype(np.float64)
c, r, d = t[:, 2], t[:, 3], t[:, 8]
t0 = c[c > 0].min(); us = lambda v: (v - t0) / 1e3
names = {1: "span", 2: "couple", 3: "flatup", 4: "flatdn"}
last = int(np.argmax(d))
chain = [last]
while plan[chain[-1]]["deps"]:
    chain.append(max(plan[chain[-1]]["deps"], key=lambda x: d[x]))
for q in reversed(chain):
    p = plan[q]
    md = max([us(d[x]) for x in p['deps']], default=0)
    print(f"q{q:4d} {names[p['type']]:6s} cta {p['cta']:3d} est_fin {p['fin']:5.1f} claim {us(c[q]):6.2f} ready {us(r[q]):6.2f} done {us(d[q]):6.2f} ndeps {len(p['deps']):3d} maxdep {md:6.2f}")
    for x in sorted(x for x in plan if plan[x]["cta"] == p["cta"]):
        if x == q: break
        mdx = max([us(d[y]) for y in plan[x]['deps']], default=0)
        print(f"        before: q{x:4d} {names[plan[x]['type']]:6s} claim {us(c[x]):6.2f} ready {us(r[x]):6.2f} done {us(d[x]):6.2f} maxdep {mdx:6.2f}")
