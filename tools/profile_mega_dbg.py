"""Run a few persistent-kernel matvecs of data/cfg<k>.npz with H2B_OPT_DEBUG bits (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
k = int(sys.argv[1]); dbg = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
op = H2Operator(pk)
_abi.check(_abi.lib().h2b_set_option(op.handle, 4, dbg))
_abi.check(_abi.lib().h2b_set_option(op.handle, 1, 0))  # no graph: ncu sees plain launches
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
for _ in range(reps): op.matvec_perm(x, out=y)
torch.cuda.synchronize(); print("ok")
