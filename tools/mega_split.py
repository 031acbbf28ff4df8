"""Time the persistent kernel with far-field or near-field task bodies skipped (profiling aid)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
L = _abi.lib()
for k in [int(a) for a in sys.argv[1:]] or [1, 2]:
    sys.path.insert(0, "."); from bench import load; pk, ex = load(k)
    op = H2Operator(pk)
    _abi.check(L.h2b_prepare_handle(op.handle))
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda(); y = torch.empty_like(x)
    from paper_1703_01175_b200.timing import L2Flusher
    flush = L2Flusher("cuda")
    res = {}
    modes = [(0, "full"), (2, "near alone"), (4, "far alone"), (1, "near + far skeleton"), (5, "far skeleton")]
    modes += [(int(a), f"dbg{a}") for a in os.environ.get("EXTRA_DEBUG", "").split(",") if a]
    for dbg, name in modes:
        _abi.check(L.h2b_set_option(op.handle, 4, dbg))
        for _ in range(3): op.matvec_perm(x, out=y)
        tot = 0.0
        for _ in range(20):
            flush.flush()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); op.matvec_perm(x, out=y); e.record(); torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        res[name] = tot / 20 * 1e3
    _abi.check(L.h2b_set_option(op.handle, 4, 0))
    nb = pk.near_bytes()
    print(f"cfg{k}: " + "  ".join(f"{n} {v:.1f} us" for n, v in res.items()) +
          f"  | near alone {nb / res['near alone'] / 1e3:.0f} GB/s")
