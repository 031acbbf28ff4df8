"""Run every golden fixture through the GPU matvec, report schedule and errors (dev aid)."""
import sys, os, glob, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi

def q(op, what):
    v = C.c_int64(); _abi.check(_abi.lib().h2b_query(op.handle, what, C.byref(v))); return v.value

for path in sorted(glob.glob("tests/golden/*.npz")) + sorted(glob.glob("data/cfg*.npz")):
    for mega in (1, 0):
        try:
            pk, ex = load_packed(path, with_extra=True)
            op = H2Operator(pk)
            _abi.check(_abi.lib().h2b_set_option(op.handle, 2, mega))
            _abi.check(_abi.lib().h2b_prepare_handle(op.handle), "prepare")
            errs = []
            for rep in range(3):
                y = op.matvec(ex["x"][:, rep % ex["x"].shape[1]])
                ref = ex["y"][:, rep % ex["x"].shape[1]]
                errs.append(np.linalg.norm(y - ref) / np.linalg.norm(ref))
            print(f"{os.path.basename(path):22s} mega={q(op,6)} tasks={q(op,7)} grid={q(op,8)} tiers={q(op,9)} "
                  f"span={q(op,2)} launches={q(op,1)} err={max(errs):.2e} dev_error={q(op,10)}", flush=True)
            op.close()
        except Exception as e:
            print(f"{os.path.basename(path)} mega={mega} FAILED: {e}", flush=True)
