"""Per-item error report of the grouped GEMM kernel vs the CPU plan interpreter (debug aid)."""
import os
import sys
import types

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_grouped_gemm import _random_plan  # noqa: E402
from oracle.plan_exec import NumpyPlanEngine  # noqa: E402
from paper_1703_01175_b200.dist import CudaPlanEngine  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(100 + q)
n_rows, q_rows = 64 * 40, 600
pays, items, segs = _random_plan(rng, 40, n_rows, q_rows)
plan = types.SimpleNamespace(payloads=pays, phases={ph: (np.array([items.size], dtype=np.int64), items, segs) for ph in range(5)})
X = rng.standard_normal((q_rows, q)) + 1j * rng.standard_normal((q_rows, q))
YH = rng.standard_normal((q_rows, q)) + 1j * rng.standard_normal((q_rows, q))
Y0 = rng.standard_normal((n_rows, q)) + 1j * rng.standard_normal((n_rows, q))
ref = [torch.from_numpy(a.copy()) for a in (X, YH, Y0)]
NumpyPlanEngine(plan).run(4, ref[0], ref[1], ref[2], q)
dev = [torch.from_numpy(a.copy()).cuda() for a in (X, YH, Y0)]
eng = CudaPlanEngine(plan, 0)
eng.run(4, dev[0], dev[1], dev[2], q)
torch.cuda.synchronize()
got, exp = dev[2].cpu().numpy(), ref[2].numpy()
bad_any = False
for n, it in enumerate(items):
    r0, m = int(it["c_row"]), int(it["m"])
    e = np.linalg.norm(got[r0:r0 + m] - exp[r0:r0 + m]) / max(np.linalg.norm(exp[r0:r0 + m]), 1e-300)
    sg = segs[it["seg0"]:it["seg0"] + it["nseg"]]
    bad_rows = np.nonzero(np.abs(got[r0:r0 + m] - exp[r0:r0 + m]).max(1) > 1e-10)[0]
    bad_cols = np.nonzero(np.abs(got[r0:r0 + m] - exp[r0:r0 + m]).max(0) > 1e-10)[0]
    if e < 1e-12:
        continue
    print(n, "acc", int(it["flags"]) >> 8, "m", m, "nseg", it["nseg"], "ks", [int(s["k"]) for s in sg], "trans", [int(s["flags"]) >> 8 & 1 for s in sg][:1],
          f"err {e:.2e}", "bad rows", bad_rows[:8].tolist(), "bad cols", bad_cols[:10].tolist())
