"""GMRES(m) solve time at full size on a structure-exact operator (fixed iteration count).

python tools/gmres_big.py <cfg> <restart> <iterations>
The seeded far-field values make convergence meaningless, so the solve runs a fixed number of
Arnoldi steps (tol below reach) — e.g. 567, the CPU oracle's GMRES(50) count on the
reference-built cfg3 (tests/golden/cfg3_gmres.json) — and reports the device solve time.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1703_01175_b200 import H2Operator, gmres_solve  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

k, m, iters = (int(a) for a in sys.argv[1:4])
path = os.path.join(ROOT, "fixtures", f"cfg{k}_structure.npz")
if not os.path.exists(path):
    path = os.path.join(ROOT, "structures", f"cfg{k}.npz")
pk = load_packed(path, near_on_host=False, far_on_host=False)
op = H2Operator(pk)
rng = np.random.default_rng(0)
b = rng.standard_normal(pk.n) + 1j * rng.standard_normal(pk.n)
gmres_solve(op, b, tol=1e-15, restart=m, max_iter=min(iters, 2 * m))  # warm-up: graphs, workspace
x, rep = gmres_solve(op, b, tol=1e-15, restart=m, max_iter=iters)
out = {"cfg": k, "N": pk.n, "restart": m, "iterations": rep.iterations, "solve_s": rep.wall_time,
       "ms_per_iteration": rep.wall_time / rep.iterations * 1e3,
       "operator": f"cfg{k} structure-exact (reference block structure, seeded far field)",
       "note": "fixed iteration count (convergence of seeded values is meaningless)"}
print(json.dumps(out))
