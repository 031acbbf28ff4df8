"""Where the q=1 step's time outside its two kernels goes: event-timed cold steps with parts of
the step switched off (H2B_OPT_DEBUG bits: 2 no far kernel, 4 no near kernel, 8 no y memset;
results are then wrong).  Development aid.  Usage: python tools/overhead_probe.py [2]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import load  # noqa: E402
from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402
from paper_1703_01175_b200.timing import L2Flusher  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pk, ex = load(k)
fl = L2Flusher("cuda")
names = {0: "memset + near + far", 8: "near + far (no memset)", 2: "memset + near", 10: "near",
         4: "memset + far", 12: "far", 6: "memset only", 14: "empty graph"}
sel = [int(v) for v in os.environ.get("PROBE_MODES", "").split(",") if v] or list(names)
for graphs in (1,):
    for dbg in sel:
        nm = names[dbg]
        op = H2Operator(pk)
        L = _abi.lib()
        _abi.check(L.h2b_set_option(op.handle, _abi.OPT_GRAPHS, graphs))
        _abi.check(L.h2b_set_option(op.handle, _abi.OPT_DEBUG, dbg))
        x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
        y = torch.empty_like(x)
        for _ in range(5):
            op.matvec_perm(x, out=y)
        ts, sp = [], []
        L.h2b_stamp_ns.argtypes = [C.c_void_p, C.c_void_p]
        stamps = torch.zeros(2, dtype=torch.int64, device="cuda")
        cur = torch.cuda.current_stream().cuda_stream
        for it in range(120):
            fl.flush()
            _abi.check(L.h2b_spin_ns(20000, torch.cuda.current_stream().cuda_stream))
            if it % 2:  # odd iterations: %globaltimer stamps from one-thread kernels around the step
                # (the event timer ticks every ~2 us here; the stamps add a constant launch gap)
                _abi.check(L.h2b_stamp_ns(stamps.data_ptr(), cur))
                op.matvec_perm(x, out=y)
                _abi.check(L.h2b_stamp_ns(stamps.data_ptr() + 8, cur))
                torch.cuda.synchronize()
                st = stamps.cpu().numpy()
                sp.append((st[1] - st[0]) / 1e3)
                continue
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            op.matvec_perm(x, out=y)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        print(f"graphs={graphs} {nm:26s} events: mean {np.mean(ts):6.2f} us  median {np.median(ts):6.1f}  min {np.min(ts):6.1f}"
              f" | stamps: mean {np.mean(sp):6.2f}  median {np.median(sp):6.2f}  min {np.min(sp):6.2f}")
        if os.environ.get("PROBE_HIST"):
            v, c = np.unique(np.round(ts, 1), return_counts=True)
            print("   ", ", ".join(f"{a:.1f}x{b}" for a, b in zip(v, c)))
        op.close()
