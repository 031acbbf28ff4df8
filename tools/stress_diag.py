"""On a persistent-kernel mismatch, express the error on the bad rows in terms of the
near-field and far-field parts of the correct result (which contribution was lost/doubled)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
a = H2Operator(pk); b = H2Operator(pk)
_abi.check(L.h2b_set_option(b.handle, _abi.OPT_MEGA, 0))
g = torch.Generator(device="cuda"); g.manual_seed(1)
n = pk.n
V = torch.randn(40, n, dtype=torch.complex128, device="cuda", generator=g)
y = torch.zeros(n, dtype=torch.complex128, device="cuda")
prev = None
shown = 0
for it in range(3000):
    i = it % 39
    a.matvec_perm(V[i], out=y)
    yb = b.matvec_perm(V[i])
    d = (y - yb)
    if (torch.linalg.norm(d) / torch.linalg.norm(yb)).item() > 1e-13:
        yn = torch.zeros_like(y); yf = torch.zeros_like(y)
        _abi.check(L.h2b_matvec_phase(b.handle, 0, C.c_void_p(V[i].data_ptr()), C.c_void_p(yn.data_ptr()), 1, None))
        _abi.check(L.h2b_matvec_phase(b.handle, 1, C.c_void_p(V[i].data_ptr()), C.c_void_p(yf.data_ptr()), 1, None))
        torch.cuda.synchronize()
        rows = torch.nonzero(d.abs() > 1e-12 * yb.abs().max()).flatten()
        A = torch.stack([yn[rows], yf[rows]], 1).cpu().numpy()
        if prev is not None:
            A = np.concatenate([A, prev[rows.cpu().numpy()][:, None]], 1)
        coef, res, *_ = np.linalg.lstsq(A, d[rows].cpu().numpy(), rcond=None)
        r = np.linalg.norm(A @ coef - d[rows].cpu().numpy()) / np.linalg.norm(d[rows].cpu().numpy())
        print(f"it {it}: rows {rows[0].item()}..{rows[-1].item()} ({rows.numel()}), coef near/far/prev-y "
              f"{np.round(coef, 4).tolist()}, fit residual {r:.1e}")
        shown += 1
        if shown >= 12: break
    prev = y.cpu().numpy().copy()
    if it % 3 == 0:
        V[i + 1].copy_(yb / torch.linalg.norm(yb))
