"""Quick CUDA-event timing of the matvec on data/cfg<k>.npz (development aid)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import as_operator, load_packed, _abi

def q(op, what):
    v = C.c_int64(); _abi.check(_abi.lib().h2b_query(op.handle, what, C.byref(v))); return v.value

def timeit(fn, reps, flush=None):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    if flush is None:
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
    for _ in range(reps):
        flush.flush()
        s.record(); fn(); e.record(); torch.cuda.synchronize(); tot += s.elapsed_time(e)
    return tot / reps

for k in [int(a) for a in sys.argv[1:]] or [1, 2]:
    from bench import load
    pk, ex = load(k)
    t = time.time(); op = as_operator(pk); _abi.check(_abi.lib().h2b_prepare_handle(op.handle)); torch.cuda.synchronize(); tu = time.time() - t
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    y = torch.empty_like(x)
    from paper_1703_01175_b200.timing import L2Flusher
    flush = L2Flusher("cuda")
    for _ in range(5): op.matvec_perm(x, out=y)
    torch.cuda.synchronize()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ph = lambda p: _abi.lib().h2b_matvec_phase(op.handle, p, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1, st)
    warm = timeit(lambda: op.matvec_perm(x, out=y), 50)
    cold = timeit(lambda: op.matvec_perm(x, out=y), 20, flush)
    near_c = timeit(lambda: ph(0), 20, flush)
    far_c = timeit(lambda: ph(1), 20, flush)
    op.matvec_perm(x, out=y)
    B = pk.algorithmic_bytes()
    yp = y.cpu().numpy(); yy = np.empty_like(yp); yy[pk.perm] = yp
    err = np.linalg.norm(yy - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0]) if "y" in ex else float("nan")
    print(f"cfg{k}: N={pk.n} prep {tu:.2f}s span_mode={q(op,2)} ls={q(op,3)} top_staged={q(op,4)} launches={q(op,1)} | "
          f"warm {warm*1e3:.1f} us ({B/warm/1e6:.0f} GB/s) cold {cold*1e3:.1f} us ({B/cold/1e6:.0f} GB/s) | "
          f"near cold {near_c*1e3:.1f} us ({pk.near_bytes()/near_c/1e6:.0f} GB/s) far(no-graph) cold {far_c*1e3:.1f} us | relerr {err:.2e}", flush=True)
