import torch, sys
sys.path.insert(0, "/root/repo")
from paper_1703_01175_b200.timing import L2Flusher
fl = L2Flusher("cuda")
for mb in (25, 50, 100, 200, 400, 1600):
    a = torch.empty(mb * (1 << 20) // 8, dtype=torch.float64, device="cuda").fill_(1.0)
    for _ in range(3): a.sum()
    tot = 0
    for _ in range(10):
        fl.flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); a.sum(); e.record(); torch.cuda.synchronize(); tot += s.elapsed_time(e)
    ms = tot / 10
    print(f"{mb} MiB read-reduce: {ms*1e3:.1f} us -> {mb*(1<<20)/ms/1e6:.0f} GB/s")
