"""Persistent kernel launched back to back (no other kernels in between) vs stored results."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
mode = sys.argv[3] if len(sys.argv) > 3 else "alone"
pk = load_packed(f"data/cfg{k}.npz")
a = H2Operator(pk); b = H2Operator(pk)
_abi.check(L.h2b_set_option(b.handle, _abi.OPT_MEGA, 0))
g = torch.Generator(device="cuda"); g.manual_seed(1)
V = torch.randn(40, pk.n, dtype=torch.complex128, device="cuda", generator=g)
ref = torch.stack([b.matvec_perm(V[i]) for i in range(40)])
Y = torch.zeros_like(V)
bad = 0
for it in range(iters):
    i = it % 40
    a.matvec_perm(V[i], out=Y[i])
    if mode == "interleave":
        b.matvec_perm(V[(i + 7) % 40])
    if i == 39:
        d = (torch.linalg.norm(Y - ref, dim=1) / torch.linalg.norm(ref, dim=1))
        bad += int((d > 1e-13).sum())
print(f"cfg{k} {mode}: {iters} launches, mismatches {bad}")
