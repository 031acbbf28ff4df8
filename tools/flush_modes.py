"""Cold-cache timing of the matvec under different L2 flush methods (methodology check)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes as C
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
op = H2Operator(pk)
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
r = torch.zeros((256 << 20) // 8, dtype=torch.float64, device="cuda")
modes = {
    "none": lambda: None,
    "memset": lambda: w.zero_(),
    "memset+read": lambda: (w.zero_(), r.sum()),
    "read": lambda: r.sum(),
    "memset+sleep": lambda: (w.zero_(), torch.cuda._sleep(2_000_000)),
    "memset+read+sleep": lambda: (w.zero_(), r.sum(), torch.cuda._sleep(2_000_000)),
}
def run(fn, phase=None):
    tot = []
    for it in range(25):
        fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if phase is None:
            op.matvec_perm(x, out=y)
        else:
            _abi.check(L.h2b_matvec_phase(op.handle, phase, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1, None))
        e.record(); torch.cuda.synchronize()
        if it >= 5: tot.append(s.elapsed_time(e) * 1e3)
    tot.sort()
    return tot[len(tot) // 2]
for m, fn in modes.items():
    print(f"cfg{k} flush={m:18s} mega {run(fn):6.1f} us", flush=True)
