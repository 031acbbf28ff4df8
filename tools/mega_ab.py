"""q=1 step time (cold L2) with the persistent far field (OPT_MEGA=1) vs the per-phase kernels
(OPT_MEGA=0), and parity against the reference outputs.  Development aid.
Usage: python tools/mega_ab.py [cfg1 ...]"""
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

flush = L2Flusher("cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name in sys.argv[1:] or ["cfg1"]:
    pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    ref = ex["y"][:, 0]
    for mega in (1, 0):
        op = H2Operator(pk, device=0)
        _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_MEGA, mega))
        y = torch.empty_like(x)
        for _ in range(3):
            op.matvec_perm(x, out=y)
        torch.cuda.synchronize()
        yy = np.empty(pk.n, dtype=np.complex128)
        yy[pk.perm] = y.cpu().numpy()
        err = np.linalg.norm(yy - ref) / np.linalg.norm(ref)
        ts = []
        for _ in range(30):
            flush.flush()
            torch.cuda._sleep(2_000_000)
            s.record()
            op.matvec_perm(x, out=y)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        print(f"{name} mega={mega}: step {np.mean(ts[3:]):.1f} us, relerr {err:.2e}", flush=True)
        op.close()
