"""Stress the persistent kernel: many launches with varying inputs vs the multi-kernel path.
usage: stress_mega.py K [graphs(0/1)] [iters]"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
graphs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 400
dbg = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sys.path.insert(0, "."); from bench import load; pk, ex = load(k)
a = H2Operator(pk); b = H2Operator(pk)
_abi.check(L.h2b_set_option(a.handle, _abi.OPT_GRAPHS, graphs))
_abi.check(L.h2b_set_option(a.handle, 4, dbg))
_abi.check(L.h2b_set_option(b.handle, _abi.OPT_MEGA, 0))  # reference path: multi-kernel
g = torch.Generator(device="cuda"); g.manual_seed(1)
n = pk.n
leaves = np.asarray(pk.level_ptr)
lv0, lv1 = int(pk.level_ptr[-2]), int(pk.level_ptr[-1])
starts = np.asarray(pk.c_start[lv0:lv1]); sizes = np.asarray(pk.c_size[lv0:lv1])
V = torch.randn(40, n, dtype=torch.complex128, device="cuda", generator=g)
yout = torch.zeros(n, dtype=torch.complex128, device="cuda")
bad = 0; worst = 0.0; hist = {}
for it in range(iters):
    i = it % 39
    ya = a.matvec_perm(V[i], out=yout)
    yb = b.matvec_perm(V[i])
    err = (ya - yb).abs().cpu().numpy()
    d = np.linalg.norm(err) / torch.linalg.norm(yb).item()
    worst = max(worst, d)
    if d > 1e-13:
        bad += 1
        rows = np.nonzero(err > 1e-10 * np.abs(yb.cpu().numpy()).max())[0]
        lf = np.searchsorted(starts, rows, side="right") - 1
        u = np.unique(lf)
        if bad <= 6:
            print(f"it {it}: rel {d:.2e}, {rows.size} rows, leaves {u[:20].tolist()}{'...' if u.size > 20 else ''}")
        for l in u: hist[int(l)] = hist.get(int(l), 0) + 1
    if it % 3 == 0:
        V[i + 1].copy_(yb / torch.linalg.norm(yb))
e = C.c_int64(); _abi.check(L.h2b_query(a.handle, _abi.Q_DEVICE_ERROR, C.byref(e)))
print(f"cfg{k} graphs={graphs} debug={dbg}: {iters} launches, mismatches {bad}, worst rel diff {worst:.2e}, device error {e.value}")
print("leaf hit counts:", sorted(hist.items(), key=lambda t: -t[1])[:30])
q = C.c_int64()
for name, code in [("grid", _abi.Q_MEGA_GRID), ("tasks", _abi.Q_MEGA_TASKS), ("tiers", _abi.Q_MEGA_TIERS)]:
    _abi.check(L.h2b_query(a.handle, code, C.byref(q))); print(name, q.value)
print("n", n, "leaves", lv1 - lv0, "leaf sizes", np.unique(sizes))
