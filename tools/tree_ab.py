"""A/B of the q=1 far field: subtree programs (h2b_tree.cu) vs the task-graph kernel (k_mega).

For each operator: parity of both against the reference's own matvec output, cold-L2 step time
(CUDA events, L2 flushed before each call), the far-field kernel alone (near-field launch
skipped: H2B_OPT_DEBUG bit 2, timing only) and the device error word.  Development aid.
Usage: python tools/tree_ab.py [cfg1 cfg2 golden:<name> ...]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import _abi  # noqa: E402
from paper_1703_01175_b200.h2op import H2Operator  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402
from paper_1703_01175_b200.timing import L2Flusher  # noqa: E402


def q(op, what):
    v = C.c_int64()
    _abi.check(_abi.lib().h2b_query(op.handle, what, C.byref(v)))
    return v.value


def load(name):
    if name.startswith("golden:"):
        return load_packed(os.path.join(ROOT, "tests", "golden", name[7:] + ".npz"), with_extra=True)
    return load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)


def timed(fn, reps, flush):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        flush.flush()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.mean(ts[2:]))  # event times are quantised (~2 us): a mean, not a median


flush = L2Flusher("cuda")
for name in sys.argv[1:] or ["cfg2"]:
    pk, ex = load(name)
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    ref = ex["y"][:, 0]
    for tree in (1, 0):
        op = H2Operator(pk, device=0)
        _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_TREE, tree))
        y = torch.empty_like(x)
        for _ in range(3):
            op.matvec_perm(x, out=y)
        torch.cuda.synchronize()
        yy = np.empty(pk.n, dtype=np.complex128)
        yy[pk.perm] = y.cpu().numpy()
        err = np.linalg.norm(yy - ref) / np.linalg.norm(ref)
        t = timed(lambda: op.matvec_perm(x, out=y), 30, flush)
        # repeatability: bitwise over 20 calls
        same = True
        y0 = y.clone()
        for _ in range(20):
            op.matvec_perm(x, out=y)
            same &= bool(torch.equal(y, y0))
        _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, 4))  # far field only
        tf = timed(lambda: op.matvec_perm(x, out=y), 30, flush)
        _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, 2))  # near field only
        tn = timed(lambda: op.matvec_perm(x, out=y), 30, flush)
        _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, 0))
        tr = q(op, _abi.Q_TREE)
        print(f"{name} tree={tree} (progs {tr & 0xffff} ls {(tr >> 16) & 255} lt {(tr >> 24) & 63} flat {(tr >> 30) & 1}) relerr {err:.2e} "
              f"repeatable {same} step {t:.1f} us far-only {tf:.1f} us near-only {tn:.1f} us "
              f"B_alg/step {pk.algorithmic_bytes() / t / 1e3:.0f} GB/s err {q(op, _abi.Q_DEVICE_ERROR)} near stages {q(op, _abi.Q_NEAR_STAGES)}",
              flush=True)
        op.close()
