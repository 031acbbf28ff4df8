"""Where the host-buffer matvec's wall time goes (cfg2): H2D, D2H, device graph, whole call."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import load  # noqa: E402
from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402

pk, ex = load(2)
op = H2Operator(pk)
L = _abi.lib()
xh = torch.from_numpy(ex["x"][:, 0].copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = torch.empty_like(xh, device="cuda")
yd = torch.empty_like(xd)


def wall(fn, n=200):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return np.median(ts) * 1e6


st = torch.cuda.current_stream()
print(f"H2D 1 MiB pinned + sync: {wall(lambda: (xd.copy_(xh, non_blocking=True), torch.cuda.synchronize())):.1f} us")
print(f"D2H 1 MiB pinned + sync: {wall(lambda: (yh.copy_(yd, non_blocking=True), torch.cuda.synchronize())):.1f} us")
mv = lambda: _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), 1,  # noqa: E731
                                          C.c_void_p(st.cuda_stream)))
print(f"device matvec (graph) + sync: {wall(lambda: (mv(), torch.cuda.synchronize())):.1f} us")
print(f"h2b_matvec_host (whole call): {wall(lambda: _abi.check(L.h2b_matvec_host(op.handle, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1))):.1f} us")
print(f"empty sync: {wall(lambda: torch.cuda.synchronize()):.1f} us")
