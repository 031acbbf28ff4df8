"""Throughput on the structure-exact BASELINE cfg4 / cfg5 operators (structures/cfg<k>.npz).

python tools/bench_big.py <cfg> [q ...]  -> one JSON line per q
Operator: the reference's own cluster tree and block partition, proxy ranks, seeded V/T/S
generated in HBM, near-field sampled on the device from the geometry (tools/make_structures.py).
No parity claim (no reference output exists); checked: linearity and bitwise repeatability.
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

HBM, FP64 = 6532.5e9, 37.1e12
k = int(sys.argv[1])
qs = [int(a) for a in sys.argv[2:]] or [1]
t0 = time.time()
pk = load_packed(os.path.join(ROOT, "structures", f"cfg{k}.npz"), near_on_host=False, far_on_host=False)
dev = torch.device("cuda:0")
free0, total = torch.cuda.mem_get_info(0)
op = H2Operator(pk, device=0)
L = _abi.lib()
if pk.num_clusters > 20000:
    _abi.check(L.h2b_set_option(op.handle, _abi.OPT_MEGA, 0))
_abi.check(L.h2b_prepare_handle(op.handle))
torch.cuda.synchronize()
t_setup = time.time() - t0
st = torch.cuda.current_stream()
for q in qs:
    g = torch.Generator(device="cuda:0").manual_seed(q)
    x = torch.randn((pk.n, q), dtype=torch.complex128, device=dev, generator=g)
    if q == 1:
        x = x[:, 0].contiguous()
    y = torch.empty_like(x)
    f = lambda xx, yy: _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(xx.data_ptr()),  # noqa: E731
                                                    C.c_void_p(yy.data_ptr()), q, C.c_void_p(st.cuda_stream)))
    for _ in range(3):
        f(x, y)
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        f(x, y)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    y1 = y.clone()
    f(x, y)
    x2 = 2.0 * x
    y2 = torch.empty_like(x)
    f(x2, y2)
    torch.cuda.synchronize()
    rep = bool(torch.equal(y, y1))
    lin = float(torch.linalg.norm(y2 - 2.0 * y1) / torch.linalg.norm(y1))
    B, F = pk.algorithmic_bytes(q), pk.flops(q)
    out = {"cfg": k, "q": q, "N": pk.n, "ms": ms, "unknowns_rhs_per_s": pk.n * q / (ms * 1e-3),
           "alg_bytes": B, "flops": F, "hbm_gbs": B / (ms * 1e-3) / 1e9, "hbm_frac": B / (ms * 1e-3) / HBM,
           "tflops": F / (ms * 1e-3) / 1e12, "fp64_frac": F / (ms * 1e-3) / FP64,
           "device_bytes": op.device_bytes(), "gpu_mem_total": total, "setup_s": t_setup,
           "bitwise_repeatable": rep, "linearity_rel": lin,
           "operator": f"cfg{k} structure-exact (reference tree/blocks, proxy ranks, seeded V/T/S, "
                       "near-field sampled on device)"}
    print(json.dumps(out), flush=True)
    del x, y, y1, x2, y2
