"""Breakdown of the end-to-end drop-in call matvec(h2, x) on numpy buffers (development aid)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import _abi, as_operator, matvec  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

pk, ex = load_packed(os.path.join(ROOT, "fixtures", "cfg2.npz"), with_extra=True)
op = as_operator(pk)
L = _abi.lib()
x = ex["x"][:, 0].copy()
y = np.empty_like(x)
xh = torch.from_numpy(x.copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
for _ in range(5):
    matvec(pk, x)


def med(f, n=60):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6


print(f"matvec(pk, x) numpy            {med(lambda: matvec(pk, x)):7.1f} us")
print(f"op.matvec(x)                   {med(lambda: op.matvec(x)):7.1f} us")
print(f"C-ABI pageable x, y            {med(lambda: L.h2b_matvec_host(op.handle, x.ctypes.data, y.ctypes.data, 1)):7.1f} us")
print(f"C-ABI pinned x, y              {med(lambda: L.h2b_matvec_host(op.handle, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1)):7.1f} us")
print(f"np.empty_like(x)               {med(lambda: np.empty_like(x)):7.1f} us")
print(f"np.empty_like + fill           {med(lambda: np.empty_like(x).fill(0)):7.1f} us")
print(f"memcpy 1 MiB numpy->numpy      {med(lambda: np.copyto(y, x)):7.1f} us")
