"""Pin the cfg3 GMRES(50) iteration count with the CPU restatement (slow: ~15 min).

Writes tests/golden/cfg3_gmres.json: iterations / history length / converged of
oracle.krylov_oracle.gmres_solve on the reference-built cfg3 operator with the seeded
plane-wave RHS (SURVEY.md §8d cfg 3), solved in the permuted space.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import h2_oracle as ho  # noqa: E402
from oracle import krylov_oracle as ko  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

pk, ex = load_packed(os.path.join(ROOT, "data", "cfg3.npz"), with_extra=True)
b = ex["rhs_plane_wave"][pk.perm]
t = time.time()
x, rep = ko.gmres_solve(lambda v: ho.matvec_perm_packed(pk, v), b, tol=1e-6, restart=50, max_iter=3000)
out = dict(config="cfg3 plate 512^2, GMRES(50) to 1e-6, x0 = 0, seeded plane-wave RHS",
           iterations=rep.iterations, converged=rep.converged, history_last=rep.residual_history[-3:],
           cpu_seconds=time.time() - t, matvec="oracle.h2_oracle.matvec_perm_packed")
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "cfg3_gmres.json"), "w"), indent=1)
print(out)
