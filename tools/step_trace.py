"""Timeline of one whole q=1 matvec step (tree far field + near stream, both traced), cold L2.

Stamps of both kernels (globaltimer ns) relative to the earliest kernel entry, median over 8
calls, next to the event-timed step (same calls).  Development aid.
Usage: python tools/step_trace.py [cfg2]
"""
import ctypes as C
import os
import sys

os.environ.setdefault("H2B_NEAR_TRACE", "1")
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
pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True)
op = H2Operator(pk, device=0)
x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
y = torch.empty_like(x)
if os.environ.get("STEP_DEBUG"):
    _abi.check(_abi.lib().h2b_set_option(op.handle, _abi.OPT_DEBUG, int(os.environ["STEP_DEBUG"])))
op.matvec_perm(x, out=y)
L = _abi.lib()
L.h2b_near_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
L.h2b_tree_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
v = C.c_int64()
_abi.check(L.h2b_query(op.handle, _abi.Q_TREE, C.byref(v)))
nprog = v.value & 0xffff
if int(os.environ.get("STEP_DEBUG", "0")) & 2:
    nprog = 0  # no far kernel: its stamps are stale
v2 = C.c_int64()
_abi.check(L.h2b_query(op.handle, _abi.Q_NEAR_SMEM, C.byref(v2)))
v3 = C.c_int64()
_abi.check(L.h2b_query(op.handle, _abi.Q_NEAR_STAGES, C.byref(v3)))
print(f"tree programs {nprog}, tree smem {v.value >> 32} B, near smem {v2.value} B, near stages {v3.value}")
ncta = int(os.environ.get("H2B_NEAR_GRID", torch.cuda.get_device_properties(0).multi_processor_count))
flush = L2Flusher("cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
L.h2b_stamp_ns.argtypes = [C.c_void_p, C.c_void_p]
stamps = torch.zeros(2, dtype=torch.int64, device="cuda")
cur = torch.cuda.current_stream().cuda_stream
rows = []
for rep in range(10):
    flush.flush()
    torch.cuda._sleep(2_000_000)  # keep the host ahead of the device: launch overhead hidden
    s.record()
    _abi.check(L.h2b_stamp_ns(stamps.data_ptr(), cur))
    op.matvec_perm(x, out=y)
    _abi.check(L.h2b_stamp_ns(stamps.data_ptr() + 8, cur))
    e.record()
    torch.cuda.synchronize()
    st = stamps.cpu().numpy()
    nt = np.zeros((ncta, 24), dtype=np.int64)
    _abi.check(L.h2b_near_trace(op.handle, nt.ctypes.data, ncta))
    tt = np.zeros((nprog, 32), dtype=np.int64) if nprog else None
    if nprog:
        _abi.check(L.h2b_tree_trace(op.handle, tt.ctypes.data, nprog))
    if rep == 9 and nprog:
        far_sm = set(int(v) for v in tt[:, 15])
        near_sm = nt[:, 7]
        free = [c for c in range(ncta) if int(near_sm[c]) not in far_sm]
        print(f"near CTAs on SMs without a far program: {len(free)}: {free}")
        ex = (nt[:, 5] - min(nt[:, 0].min(), tt[:, 0][tt[:, 0] > 0].min())) / 1e3
        fs = set(free)
        a = np.array([ex[c] for c in range(ncta) if c in fs])
        b = np.array([ex[c] for c in range(ncta) if c not in fs])
        if len(a) and len(b):
            print(f"near exit (us) on SMs without a program: min {a.min():.1f} med {np.median(a):.1f} max {a.max():.1f}; "
                  f"beside a program: min {b.min():.1f} med {np.median(b):.1f} max {b.max():.1f}")
    if rep < 2:
        continue
    t0 = nt[:, 0].min()
    if nprog:
        t0 = min(t0, tt[:, 0][tt[:, 0] > 0].min())
    r = {"event_us": s.elapsed_time(e) * 1e3, "stamp.before.min": (st[0] - t0) / 1e3, "stamp.after.min": (st[1] - t0) / 1e3}
    rel = (nt[:, :6] - t0) / 1e3
    for j, nm in enumerate(["entry", "rec0", "issued_all", "landed0", "consumed_all", "exit"]):
        r[f"near.{nm}.min"] = rel[:, j].min()
        r[f"near.{nm}.med"] = np.median(rel[:, j])
        r[f"near.{nm}.max"] = rel[:, j].max()
    if nprog:
        tr = np.where(tt[:, :16] > 0, (tt[:, :16] - t0) / 1e3, np.nan)
        nb = int(np.isnan(tr[:, 2]).sum())  # bottom programs have no "ext" stamp
        for lab, sel in (("bottom", slice(0, nb)), ("top", slice(nb, nprog))):
            for j, nm in enumerate(["start", "staged", "ext", "pub_up", "cpl_wait", "dn_wait0", "dn_wait1",
                                    "down_end", "end"]):
                col = tr[sel, j]
                if np.isfinite(col).any():
                    r[f"{lab}.{nm}.min"] = np.nanmin(col)
                    r[f"{lab}.{nm}.med"] = np.nanmedian(col)
                    r[f"{lab}.{nm}.max"] = np.nanmax(col)
    rows.append(r)
keys = rows[0].keys()
med = {k: float(np.median([r[k] for r in rows if k in r])) for k in keys}
print(f"{name}: event-timed step {med['event_us']:.1f} us; stamps in us from the first kernel entry (min/median/max over CTAs, median of 8 calls)")
groups = {}
for k, val in med.items():
    if k == "event_us":
        continue
    base, stat = k.rsplit(".", 1)
    groups.setdefault(base, {})[stat] = val
for base, st in groups.items():
    print(f"  {base:22s} {st.get('min', float('nan')):7.2f} {st.get('med', float('nan')):7.2f} {st.get('max', float('nan')):7.2f}")
op.close()
