"""Multi-RHS matvec throughput (q columns) on the FP64 tensor pipe vs the CUDA-core path.

python tools/bench_mrhs.py [cfg] [q ...]   -> one JSON line per q
F(q) = 8 q (2E_V + 2E_T + E_S + E_D) useful real flops; the FP64 peak is the
measured DMMA/DFMA throughput of tools/micro/dmma_bench.cu (37.1 TFLOP/s on B200).
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import load  # noqa: E402
from paper_1703_01175_b200 import H2Operator, _abi  # noqa: E402

FP64_PEAK = 37.1e12
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
qs = [int(a) for a in sys.argv[2:]] or [64]
pk, ex = load(cfg)
op = H2Operator(pk)
L = _abi.lib()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
for q in qs:
    g = torch.Generator().manual_seed(q)
    x = torch.complex(torch.randn(pk.n, q, generator=g, dtype=torch.float64),
                      torch.randn(pk.n, q, generator=g, dtype=torch.float64)).to(dev)
    y = torch.empty_like(x)
    res = {"cfg": cfg, "q": q, "N": pk.n, "flops": pk.flops(q)}
    for mode in (1, 0):
        _abi.check(L.h2b_set_option(op.handle, _abi.OPT_MRHS, mode))
        f = lambda: _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(x.data_ptr()),  # noqa: E731
                                                 C.c_void_p(y.data_ptr()), q, C.c_void_p(st.cuda_stream)))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        reps = 10 if mode else 2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            f()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        key = "dmma" if mode else "cuda_core"
        res[key] = {"ms": ms, "tflops": pk.flops(q) / (ms * 1e-3) / 1e12,
                    "frac_fp64_peak": pk.flops(q) / (ms * 1e-3) / FP64_PEAK,
                    "unknowns_rhs_per_s": pk.n * q / (ms * 1e-3)}
        if mode:
            y_dmma = y.clone()
    res["dmma_vs_cuda_core_rel"] = float((torch.linalg.norm(y_dmma - y) / torch.linalg.norm(y)).item())
    n_l = C.c_int64()
    _abi.check(L.h2b_query(op.handle, _abi.Q_MRHS_LAUNCHES, C.byref(n_l)))
    res["launches"] = n_l.value
    print(json.dumps(res), flush=True)
