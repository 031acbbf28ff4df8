"""Repetition stress of the q=1 persistent step (near-field stream beside the far field): many
launches on BASELINE configs, every result compared bitwise with the first one, device error
word checked.  Development aid (run under `timeout`).  Usage: python tools/stress_near.py [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import load  # noqa: E402
from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
for k in (2, 1):
    pk, ex = load(k)
    op = H2Operator(pk)
    xs = [torch.from_numpy(ex["x"][pk.perm, j].copy()).cuda() for j in range(2)]
    ys = [op.matvec_perm(x).clone() for x in xs]
    y = torch.empty_like(xs[0])
    bad = 0
    for it in range(reps):
        j = it & 1
        op.matvec_perm(xs[j], out=y)
        if it % 50 == 0:
            torch.cuda.synchronize()
        if not torch.equal(y, ys[j]):
            bad += 1
    torch.cuda.synchronize()
    v = C.c_int64()
    _abi.check(_abi.lib().h2b_query(op.handle, _abi.Q_DEVICE_ERROR, C.byref(v)))
    yh = np.empty(pk.n, dtype=np.complex128)
    yh[pk.perm] = ys[0].cpu().numpy()
    rel = np.linalg.norm(yh - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0])
    print(f"cfg{k}: {reps} launches, {bad} differ from the first, device error {v.value}, relerr {rel:.2e}", flush=True)
    op.close()
