"""Record the persistent kernel's per-task timeline on data/cfg<k>.npz (L2 flushed first)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
op = H2Operator(pk)
L = _abi.lib()
_abi.check(L.h2b_prepare_handle(op.handle))
_abi.check(L.h2b_set_option(op.handle, _abi.OPT_TRACE, 1))
n = C.c_int64(); _abi.check(L.h2b_query(op.handle, _abi.Q_MEGA_TASKS, C.byref(n)))
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): op.matvec_perm(x, out=y)
flush.zero_(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); op.matvec_perm(x, out=y); e.record(); torch.cuda.synchronize()
out = np.zeros(10 * n.value, dtype=np.int64)
_abi.check(L.h2b_get_trace(op.handle, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value))
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_cfg{k}.npy", out.reshape(-1, 10))
print(f"cfg{k}: event time {s.elapsed_time(e)*1e3:.1f} us, {n.value} tasks")
