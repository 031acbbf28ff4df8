"""A few persistent-kernel launches on data/cfg<k>.npz with H2B_OPT_DEBUG bits (for ncu captures).
usage: one_launch.py K [debug] [launches]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
from paper_1703_01175_b200.timing import L2Flusher
L = _abi.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
op = H2Operator(pk)
_abi.check(L.h2b_prepare_handle(op.handle))
_abi.check(L.h2b_set_option(op.handle, _abi.OPT_GRAPHS, 0))
_abi.check(L.h2b_set_option(op.handle, 4, dbg))
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
fl = L2Flusher("cuda")
for _ in range(n):
    fl.flush()
    op.matvec_perm(x, out=y)
torch.cuda.synchronize()
print("ok")
