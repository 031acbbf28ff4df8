"""Run every golden fixture through the GPU matvec, report schedule and errors (dev aid)."""
import sys, os, glob, ctypes as C, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi

def q(op, what):
    v = C.c_int64(); _abi.check(_abi.lib().h2b_query(op.handle, what, C.byref(v))); return v.value

for path in sorted(glob.glob("tests/golden/*.npz")) + sorted(glob.glob("data/cfg*.npz")):
    for graphs in (0, 1):
        try:
            pk, ex = load_packed(path, with_extra=True)
            op = H2Operator(pk)
            _abi.check(_abi.lib().h2b_set_option(op.handle, 1, graphs))
            _abi.check(_abi.lib().h2b_prepare_handle(op.handle), "prepare")
            y = op.matvec(ex["x"][:, 0])
            err = np.linalg.norm(y - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0])
            print(f"{os.path.basename(path)} graphs={graphs} span={q(op,2)} ls={q(op,3)} top={q(op,4)} "
                  f"launches={q(op,1)} err={err:.2e}", flush=True)
            op.close()
        except Exception as e:
            print(f"{os.path.basename(path)} graphs={graphs} FAILED: {e}", flush=True)
