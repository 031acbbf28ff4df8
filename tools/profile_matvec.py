"""Run a few matvecs of data/cfg<k>.npz (for ncu launch lists / captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import as_operator, load_packed, _abi
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
graphs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
op = as_operator(pk)
_abi.check(_abi.lib().h2b_set_option(op.handle, 1, graphs))
_abi.check(_abi.lib().h2b_prepare_handle(op.handle))
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
y = torch.empty_like(x)
for _ in range(reps):
    op.matvec_perm(x, out=y)
torch.cuda.synchronize()
print("ok", float(torch.linalg.norm(y)))
