"""Smoke-size workload for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run.

Exercises every hot kernel family once on small reference fixtures: the q=1 matvec (near-field
stream with the subtree-program far field on line2048, with the task-graph far field on cube2),
the multi-RHS DMMA path (q = 4), the fused GMRES Arnoldi cluster step and the fused BiCGStab
segments.  Results are checked against the reference outputs so a silent corruption shows.
Usage: compute-sanitizer --tool <tool> python tools/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1703_01175_b200 import H2Operator, _abi, bicgstab_solve, gmres_solve  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for name in ("line2048", "cube2"):
    pk, ex = load_packed(os.path.join(ROOT, "tests", "golden", name + ".npz"), with_extra=True)
    op = H2Operator(pk, device=0)
    import ctypes as C
    v = C.c_int64()
    _abi.check(_abi.lib().h2b_prepare_handle(op.handle))
    _abi.check(_abi.lib().h2b_query(op.handle, _abi.Q_TREE, C.byref(v)))
    t = C.c_int64()
    _abi.check(_abi.lib().h2b_query(op.handle, _abi.Q_MEGA, C.byref(t)))
    e1 = rel(op.matvec(ex["x"][:, 0]), ex["y"][:, 0])
    e2 = rel(op.matvec(ex["x"][:, 0]), ex["y"][:, 0])
    X = ex["x"][:, :2]
    Xq = np.concatenate([X, 1j * X], 1)
    eq = rel(op.matmat(Xq)[:, :2], ex["y"][:, :2])
    b = ex["x"][:, 0]
    xg, rg = gmres_solve(op, b, tol=1e-8, restart=30, max_iter=300)
    xb, rb = bicgstab_solve(op, b, tol=1e-6, max_iter=300)
    print(f"{name}: tree {v.value != 0} mega {t.value} matvec {e1:.1e} {e2:.1e} q=4 {eq:.1e} "
          f"gmres {rg.iterations} it conv {rg.converged} bicgstab {rb.iterations} it conv {rb.converged}",
          flush=True)
    assert e1 <= 1e-10 and e2 <= 1e-10 and eq <= 1e-10 and rg.converged
    op.close()
print("sanitize smoke ok")
