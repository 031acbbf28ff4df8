"""Record the persistent kernel's per-task timeline on data/cfg<k>.npz (L2 flushed first).
usage: trace_mega.py K [debug]   (debug: H2B_OPT_DEBUG bits, profiling only)"""
import sys, os, ctypes as C
os.makedirs("gpurun_out", exist_ok=True)
os.environ.setdefault("H2B_DUMP_PLAN", f"gpurun_out/plan_cfg{sys.argv[1] if len(sys.argv) > 1 else 2}.txt")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sys.path.insert(0, "."); from bench import load; pk, ex = load(k)
op = H2Operator(pk)
L = _abi.lib()
_abi.check(L.h2b_prepare_handle(op.handle))
_abi.check(L.h2b_set_option(op.handle, _abi.OPT_TRACE, 1))
_abi.check(L.h2b_set_option(op.handle, 4, dbg))
n = C.c_int64(); _abi.check(L.h2b_query(op.handle, _abi.Q_MEGA_TASKS, C.byref(n)))
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
from paper_1703_01175_b200.timing import L2Flusher
flush = L2Flusher("cuda")
for _ in range(5): op.matvec_perm(x, out=y)
flush.flush(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); op.matvec_perm(x, out=y); e.record(); torch.cuda.synchronize()
out = np.zeros(10 * n.value, dtype=np.int64)
_abi.check(L.h2b_get_trace(op.handle, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value))
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_cfg{k}{'_dbg%d' % dbg if dbg else ''}.npy", out.reshape(-1, 10))
print(f"cfg{k} debug={dbg}: event time {s.elapsed_time(e)*1e3:.1f} us, {n.value} tasks")
