"""Print the persistent-kernel configuration chosen for fixtures / configs."""
import sys, os, glob, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
paths = sys.argv[1:] or sorted(glob.glob("data/cfg[12].npz"))
for p in paths:
    op = H2Operator(load_packed(p))
    _abi.check(L.h2b_prepare_handle(op.handle))
    v = {}
    for name in ("MEGA", "MEGA_GRID", "MEGA_TASKS", "MEGA_TIERS", "MEGA_SMEM", "NEAR_TASKS", "NEAR_STAGES",
                 "NEAR_SMEM", "NEAR_VARIANT"):
        q = C.c_int64(); _abi.check(L.h2b_query(op.handle, getattr(_abi, "Q_" + name), C.byref(q))); v[name] = q.value
    print(os.path.basename(p), v, flush=True)
