"""Step time of the q=1 persistent path with one of its two concurrent kernels switched off
(H2B_OPT_DEBUG: 2 = no far-field kernel, 4 = no near-field kernel; results are then wrong).
Development aid: shows which kernel bounds the concurrent step."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)
import torch  # noqa: E402

from bench import load  # noqa: E402
from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402
from paper_1703_01175_b200.timing import L2Flusher  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pk, ex = load(k)
fl = L2Flusher("cuda")
for dbg in (0, 2, 4):
    op = H2Operator(pk)
    L = _abi.lib()
    _abi.check(L.h2b_set_option(op.handle, _abi.OPT_DEBUG, dbg))
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    y = torch.empty_like(x)
    for _ in range(5):
        op.matvec_perm(x, out=y)
    tot = 0.0
    for _ in range(20):
        fl.flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        op.matvec_perm(x, out=y)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    print({0: "both", 2: "near only", 4: "far only"}[dbg], f"{tot / 20 * 1e3:.1f} us cold")
    op.close()
