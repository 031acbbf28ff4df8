"""Block GMRES(30) solve of 64 seeded right-hand sides on cfg1 (timing / launch-list target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1703_01175_b200 import H2Operator, block_gmres_solve  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

pk, ex = load_packed(os.path.join(ROOT, "fixtures", "cfg1.npz"), with_extra=True)
op = H2Operator(pk)
rng = np.random.default_rng(64)
B = rng.standard_normal((pk.n, 64)) + 1j * rng.standard_normal((pk.n, 64))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    X, rep = block_gmres_solve(op, B, tol=1e-6, restart=30, max_iter=600)
    print(f"block GMRES(30) q=64: {rep.iterations} it, {rep.wall_time * 1e3:.1f} ms, conv {rep.converged}", flush=True)
