"""Per-program timeline of the q=1 tree far field (H2B_TREE_TRACE), far field alone, cold L2."""
import ctypes as C
import os
import sys

os.environ.setdefault("H2B_TREE_TRACE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import _abi  # noqa: E402
from paper_1703_01175_b200.h2op import H2Operator  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402
from paper_1703_01175_b200.timing import L2Flusher  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # OPT_DEBUG: 4 far only, 0 both kernels
warm = len(sys.argv) > 3 and sys.argv[3] == "warm"  # no L2 flush between calls
pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)
op = H2Operator(pk, device=0)
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
y = torch.empty_like(x)
op.matvec_perm(x, out=y)
_abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, mode))
v = C.c_int64()
_abi.check(_abi.lib().h2b_query(op.handle, _abi.Q_TREE, C.byref(v)))
n = v.value & 0xffff
flush = L2Flusher("cuda")
L = _abi.lib()
L.h2b_tree_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
names = ["start", "staged", "ext", "pub_up", "cpl_wait", "dn_wait0", "dn_wait1", "down_end", "end", "up0", "up1", "up2", "up3", "up4", "up5"]
if os.environ.get("H2B_TREE_TRACE") == "3":  # stamps 9-14 of the downward pass instead
    names[9:15] = ["xg", "couple", "dn0", "dn1", "dn2", "dn3"]
if os.environ.get("H2B_TREE_TRACE") in ("4", "5"):  # the bottom programs' last step (5: run twice)
    names[9:15] = ["-", "-", "g_in", "leaves", "leaves1", "-"]
acc = []
for rep in range(10):
    if not warm:
        flush.flush()
    op.matvec_perm(x, out=y)
    torch.cuda.synchronize()
    tr2 = np.zeros((n, 32), dtype=np.int64)
    _abi.check(L.h2b_tree_trace(op.handle, tr2.ctypes.data, n))
    tr, ck = tr2[:, :16], tr2[:, 16:]
    # globaltimer aligns the programs (start); SM clocks give the fine deltas inside a program
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    start = (tr[:, :1] - t0) / 1e3
    rel = np.where(tr > 0, start + (ck - ck[:, :1]) / 1965.0, np.nan)
    acc.append(rel)
rel = np.nanmedian(np.stack(acc), axis=0)
nb = n - int((rel[:, 2] == rel[:, 2]).sum())
print(f"{name} mode {mode} {'warm' if warm else 'cold'}: {n} programs ({nb} bottom), times in us from the first program start (median of 10)")
for label, sel in (("bottom", slice(0, nb)), ("top", slice(nb, n))):
    r = rel[sel]
    if r.size == 0:
        continue
    print(f"  {label}: " + "  ".join(f"{names[j]} {np.nanmin(r[:, j]):.1f}/{np.nanmedian(r[:, j]):.1f}/{np.nanmax(r[:, j]):.1f}"
                                    for j in ((0, 1, 2, 3, 4, 9, 10, 5, 6, 11, 12, 13, 14, 7, 8) if os.environ.get("H2B_TREE_TRACE") in ("3", "4", "5") else (0, 1, 2, 9, 10, 11, 12, 13, 14, 3, 4, 5, 6, 7, 8)) if np.isfinite(r[:, j]).any()))
if os.environ.get("H2B_TREE_TRACE") in ("3", "4"):  # slot 15: SM cycles of warp 0's first coupling colsum
    meta = tr2[:, 31]
    cyc = tr2[:, 15]
    for lab, sel in (("bottom", slice(0, nb)), ("top", slice(nb, n))):
        m = meta[sel]
        print(f"  {lab}: first coupling colsum {np.median(cyc[sel]):.0f} cycles (rows {np.median(m >> 16):.0f}, "
              f"k {np.median((m >> 8) & 255):.0f}, sh {np.median(m & 255):.0f})")
