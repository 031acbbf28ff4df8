"""Quick CUDA-event timing of the matvec on data/cfg<k>.npz (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_01175_b200 import as_operator, load_packed

for k in [int(a) for a in sys.argv[1:]] or [1, 2]:
    pk, ex = load_packed(f"data/cfg{k}.npz", with_extra=True)
    t = time.time(); op = as_operator(pk); torch.cuda.synchronize(); tu = time.time() - t
    x = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    y = torch.empty_like(x)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5): op.matvec_perm(x, out=y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # warm (back-to-back)
    s.record()
    for _ in range(50): op.matvec_perm(x, out=y)
    e.record(); torch.cuda.synchronize(); warm = s.elapsed_time(e) / 50
    # cold (L2 flushed)
    tot = 0.0
    for _ in range(20):
        flush.zero_()
        s.record(); op.matvec_perm(x, out=y); e.record(); torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    cold = tot / 20
    B = pk.algorithmic_bytes()
    yp = y.cpu().numpy(); yy = np.empty_like(yp); yy[pk.perm] = yp
    err = np.linalg.norm(yy - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0])
    print(f"cfg{k}: N={pk.n} upload {tu:.2f}s warm {warm*1e3:.1f} us ({B/warm/1e6:.0f} GB/s) "
          f"cold {cold*1e3:.1f} us ({B/cold/1e6:.0f} GB/s) relerr {err:.2e}", flush=True)
