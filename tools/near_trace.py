"""Per-CTA timeline of the near-field stream (H2B_NEAR_TRACE), cold L2.  Development aid.

Usage: python tools/near_trace.py [cfg2] [mode]   (mode = OPT_DEBUG: 2 near only, 0 both kernels)
Prints, over 10 calls, the median across CTAs (and the max) of each stamp relative to the
earliest CTA entry, the per-CTA streaming rate between the first landed and the last consumed
block, and the spread of CTA finish times.
"""
import ctypes as C
import os
import sys

os.environ.setdefault("H2B_NEAR_TRACE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import _abi  # noqa: E402
from paper_1703_01175_b200.h2op import H2Operator  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402
from paper_1703_01175_b200.timing import L2Flusher  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)
op = H2Operator(pk, device=0)
if os.environ.get("TREE") is not None:  # TREE=0: the task-graph far plan (more near stages)
    _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_TREE, int(os.environ["TREE"])))
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
y = torch.empty_like(x)
op.matvec_perm(x, out=y)
_abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, mode))
v = C.c_int64()
_abi.check(_abi.lib().h2b_query(op.handle, _abi.Q_NEAR_STAGES, C.byref(v)))
L = _abi.lib()
L.h2b_near_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
n = torch.cuda.get_device_properties(0).multi_processor_count
flush = L2Flusher("cuda")
names = ["entry", "rec0", "issued_all", "landed0", "consumed_all", "exit"]
acc, rates, spread, cyc = [], [], [], []
dbytes = pk.dbuf.nbytes if hasattr(pk, "dbuf") else 0
for rep in range(10):
    flush.flush()
    op.matvec_perm(x, out=y)
    torch.cuda.synchronize()
    t = np.zeros((n, 24), dtype=np.int64)
    _abi.check(L.h2b_near_trace(op.handle, t.ctypes.data, n))
    if rep < 2:
        continue
    t0 = t[:, 0].min()
    rel = (t[:, :6] - t0) / 1e3
    acc.append(rel)
    blocks = t[:, 6]
    dur = (t[:, 4] - t[:, 3]) / 1e3
    rates.append(np.median(blocks / np.maximum(dur, 1e-3)))
    spread.append((rel[:, 4].min(), rel[:, 4].max()))
    cyc.append(np.concatenate([t[:, 8:15], t[:, 16:18]], 1) / 1965.0)  # SM cycles -> us at the max clock
a = np.stack(acc)
print(f"{name} mode {mode}: near stages {v.value}, CTAs {n}, blocks/CTA median {np.median(blocks):.0f} "
      f"(min {blocks.min()}, max {blocks.max()}), D {dbytes / 1e6:.1f} MB")
for j, nm in enumerate(names):
    print(f"  {nm:13s} median {np.median(a[:, :, j]):7.2f} us   max {np.median(a[:, :, j].max(1)):7.2f} us")
print(f"  per-CTA rate {np.median(rates):.2f} blocks/us; last-consumed spread "
      f"{np.median([s[0] for s in spread]):.2f} .. {np.median([s[1] for s in spread]):.2f} us")
c = np.median(np.stack(cyc), axis=0)
for j, nm in enumerate(["prod: stage-free wait", "prod: record wait", "prod: rec-buffer wait", "prod: index load",
                        "cons: block wait", "cons: record wait", "cons: total", "cons: math+release", "cons: leaf ends"]):
    print(f"  {nm:24s} median {np.median(c[:, j]):7.2f} us  max {c[:, j].max():7.2f} us")
op.close()
