import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1703_01175_b200 import as_operator, matvec
from paper_1703_01175_b200.pack import load_packed
pk, ex = load_packed("fixtures/cfg2.npz", with_extra=True)
op = as_operator(pk)
x = ex["x"][:, 0].copy()
for _ in range(5): matvec(pk, x)
def med(f, n=50):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6
print("matvec(pk, x) numpy:", med(lambda: matvec(pk, x)))
print("op.matvec(x):", med(lambda: op.matvec(x)))
pin = torch.empty(pk.n, dtype=torch.complex128).pin_memory().numpy()
dst = np.empty_like(x)
print("memcpy 1 MiB pageable->pinned:", med(lambda: np.copyto(pin, x)))
print("memcpy 1 MiB pinned->pageable:", med(lambda: np.copyto(dst, pin)))
print("np.empty_like + copy:", med(lambda: np.copyto(np.empty_like(x), pin)))
