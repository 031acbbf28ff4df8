"""Multi-RHS matvec (q columns) on a fixture operator: event time per call, for ncu launch lists.
Usage: python tools/mrhs_probe.py [cfg1] [q] [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
q = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)
op = H2Operator(pk, device=0)
L = _abi.lib()
rng = np.random.default_rng(64)
B = rng.standard_normal((pk.n, q)) + 1j * rng.standard_normal((pk.n, q))
xd = torch.from_numpy(B[pk.perm]).cuda()
yd = torch.empty_like(xd)
st = torch.cuda.current_stream()


def mv():
    _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), q,
                                 C.c_void_p(st.cuda_stream)))


for _ in range(3):
    mv()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(reps):
    mv()
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
yy = np.empty_like(B)
yy[pk.perm] = yd.cpu().numpy()
print(f"{name} q={q}: {ms * 1e3:.1f} us per matmat, {pk.flops(q) / (ms * 1e-3) / 1e12:.2f} TF")
