#!/usr/bin/env python
"""Benchmark of the B200 H² matvec hot path (BASELINE.json metric).

Metric: H² matvec unknowns·RHS/s (complex128).  Workload: BASELINE config 2
(configs[1]: 1-D line of 65,536 points over 2048 λ, leaf 32, η = 1, tol 1e-4,
one complex128 N(0,1) RHS) — the operator built by the reference builder and
shipped packed as data/cfg2.npz (tools/make_golden.py).

* ``value``   whole-job unknowns/s of the device matvec, x and y resident in
              HBM, L2 flushed (256 MiB write, then 256 MiB read so no dirty lines remain) before every timed step, each
              step timed with CUDA events on the launching stream.
* ``e2e``     the same metric through the reference-facing call with HOST
              buffers (h2b_matvec_host: pinned H2D, gather, matvec, scatter,
              D2H), wall clock per call.
* ``roofline`` the whole matvec step (the near-field stream and the far-field
              task graph run concurrently, so the step is the unit one launch
              pair processes): algorithmic bytes B_alg = 16(E_V+E_T+E_S+E_D) +
              32(N+K) / the average event-timed step, against the measured HBM
              copy bandwidth in MEASURED_PEAKS.json; ``dominant_kernel`` times
              the near-field kernel alone the same way.
* ``cpu_baseline`` the reference algorithm restated on the CPU
              (oracle/h2_oracle.py, a faithful port of arith.matvec) timed on
              this host, 1 thread.
``--impl reference`` times that CPU port alone and prints the same line.
Multi-GPU (torchrun, N > 1): the headline shards right-hand sides across ranks — every rank
holds the operator and applies it to its own RHS (independent objects, no data-path collective,
weak scaling; max over ranks of the device time).  Beside it, ``partitioned_strong`` measures the
same operator partitioned by subtree over the N GPUs (paper_1703_01175_b200/dist.py: one NCCL
all-gather of x and x̂ per matvec, strong scaling of one RHS); ``--partitioned`` makes that the
headline.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the reference CPU path is single-threaded
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "H2 matvec unknowns*RHS/s (complex128)"
UNIT = "unknowns*RHS/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="h2b", choices=["h2b", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="budget of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--no-cube", action="store_true",
                    help="N > 1: skip the partitioned 2M-unknown cube (cfg4) leg")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "allgather"],
                    help="partitioned path: fused P2P exchange or NCCL all-gather")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the subtree-partitioned path even on one GPU (always on for N > 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("H2B_BENCH_ONE_GPU"):  # functional test of the N > 1 flow on one GPU (gloo)
        local = 0
    return rank, world, local


def max_over_ranks(vals, dev):
    """Element-wise max over ranks of a list of floats (device tensor under NCCL, host under gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return list(vals)
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(vals), device=on, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def config_desc(k, pk):
    names = {1: "cfg1 cube 16^3 (N=4096), leaf 32, tol 1e-4",
             2: "cfg2 line 2048 lambda at 32 pts/lambda (N=65536), leaf 32, tol 1e-4",
             3: "cfg3 plate 512^2 (N=262144), leaf 64, tol 1e-4",
             4: "cfg4 cube 128^3 (N=2097152), leaf 64, tol 1e-3",
             5: "cfg5 cube 64^3 random eps_r (N=262144), leaf 64, tol 1e-4"}
    return {"workload": names.get(k, f"cfg{k}"), "N": int(pk.n), "q": 1, "eta": 1.0,
            "operator_bytes_alg": int(pk.algorithmic_bytes()),
            "operator": (f"cfg{k} structure-exact: reference block structure/ranks, seeded V/T/S, "
                         "near-field sampled from geometry on device" if "synthetic" in pk.meta
                         else f"cfg{k}: reference block structure, far field built on the B200 by the "
                              "reference's algorithm (Stage I ACA + Stage II), near-field sampled on device"
                         if pk.meta.get("built_on_device")
                         else f"cfg{k} built by the reference h2vie builder, packed")}


def load(k):
    from paper_1703_01175_b200.pack import load_packed
    # full packed operator, else a compact copy whose near-field is re-assembled on load
    # (fixtures/ is committed for cfg1/cfg2; data/cfg3_compact.npz is shipped when present)
    for path in (os.path.join(ROOT, "data", f"cfg{k}.npz"),
                 os.path.join(ROOT, "data", f"cfg{k}_compact.npz"),
                 os.path.join(ROOT, "fixtures", f"cfg{k}.npz")):
        if os.path.exists(path):
            return load_packed(path, with_extra=True)
    # config 3: the reference block structure with the far field BUILT ON THE DEVICE from the
    # geometry (paper_1703_01175_b200.builder: the reference's Stage I / II restated, ~18 s), and
    # the reference-built operator's own matvec outputs for parity (fixtures/cfg3_ref_outputs.npz)
    sp = os.path.join(ROOT, "fixtures", f"cfg{k}_structure.npz")
    rp = os.path.join(ROOT, "fixtures", f"cfg{k}_ref_outputs.npz")
    if os.path.exists(sp) and os.path.exists(rp) and not os.environ.get("H2B_BENCH_SEEDED"):
        from paper_1703_01175_b200.builder import build_device
        from paper_1703_01175_b200.nearfield import geometry_arrays
        pk, _ = load_packed(sp, with_extra=True, near_on_host=False, far_on_host=False)
        centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
        t0 = time.perf_counter()
        pk = build_device(pk, centers, chi, k0, vol, 1e-4, 1e-4)
        ex = dict(np.load(rp))
        ex["build_s"] = time.perf_counter() - t0
        return pk, ex
    # structure-exact operator (reference block structure and ranks, seeded far-field values,
    # near-field sampled on the device): throughput only, parity is checked by the tests
    path = sp
    if not os.path.exists(path):
        return None, None
    # cfg4's far field (26 GB) is generated on the device only (no CPU path at that size)
    pk, ex = load_packed(path, with_extra=True, near_on_host=False, far_on_host=k != 4)
    rng = np.random.default_rng(0)
    ex = dict(ex, x=(rng.standard_normal((pk.n, 2)) + 1j * rng.standard_normal((pk.n, 2))))
    return pk, ex


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_port_time(pk, x, budget_s):
    """Mean seconds per matvec of the restated reference CPU path over a bounded sample."""
    from oracle import h2_oracle as ho
    if pk.dbuf.size == 0:  # structure-exact operator: the CPU path needs the near-field on host
        from paper_1703_01175_b200.nearfield import assemble_near, geometry_arrays
        pk.dbuf = assemble_near(pk, *geometry_arrays(pk.meta["geometry"]))
    ho.matvec(pk, x)  # warm
    n, t0 = 0, time.perf_counter()
    while True:
        ho.matvec(pk, x)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 1000:
            return el / n, n


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [c.strip() for c in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def gmres_bench(rank, world, local):
    """GMRES(30) to 1e-6 on BASELINE config 1 through the drop-in solver (host RHS in, host x out)."""
    if rank != 0:
        return None
    pk, ex = load(1)
    if pk is None:
        return None
    from paper_1703_01175_b200 import H2Operator, gmres_solve
    op = H2Operator(pk, device=local)
    b = ex["x"][:, 0]
    gmres_solve(op, b, tol=1e-6, restart=30, max_iter=2000)  # warm-up (graph capture, workspace)
    best = None
    for _ in range(3):
        x, rep = gmres_solve(op, b, tol=1e-6, restart=30, max_iter=2000)
        best = rep if best is None or rep.wall_time < best.wall_time else best
    res = float(np.linalg.norm(op.matvec(x) - b) / np.linalg.norm(b))
    out = {"config": "cfg1 cube 16^3 (N=4096), GMRES(30) to 1e-6, x0 = 0, N(0,1) RHS",
           "solve_s": best.wall_time, "iterations": best.iterations,
           "oracle_iterations": int(ex["gmres_iters"]) if "gmres_iters" in ex else None,
           "true_rel_residual": res, "converged": best.converged}
    op.close()
    return out


def bicgstab_bench(rank, local):
    """The reference's own solver (arith.bicgstab_solve, arith.py:605-689) at BASELINE cfg1 to
    1e-6 on the device, against the iteration count the reference itself produced."""
    if rank != 0:
        return None
    pk, ex = load(1)
    if pk is None or "bicg_iters" not in ex:
        return None
    from paper_1703_01175_b200 import H2Operator, bicgstab_solve
    op = H2Operator(pk, device=local)
    b = ex["x"][:, 0]
    bicgstab_solve(op, b, tol=1e-6, max_iter=1000)  # warm-up
    best = None
    for _ in range(3):
        x, rep = bicgstab_solve(op, b, tol=1e-6, max_iter=1000)
        best = rep if best is None or rep.wall_time < best.wall_time else best
    res = float(np.linalg.norm(op.matvec(x) - b) / np.linalg.norm(b))
    op.close()
    return {"config": "cfg1 cube 16^3, BiCGStab to 1e-6, x0 = 0, N(0,1) RHS",
            "solve_s": best.wall_time, "iterations": best.iterations,
            "reference_iterations": int(ex["bicg_iters"]), "true_rel_residual": res,
            "converged": best.converged,
            "note": "BiCGStab to 1e-6 on cfg1 is rounding-chaotic: the CPU restatement gives 121 "
                    "iterations with the reference's summation order, 124 with a batched order and "
                    "127 with the matvec scaled by (1 + 1e-15)"}


def mrhs_bench(rank, local, q=64):
    """Multi-RHS leg (BASELINE cfg5 style, 64 right-hand sides) on the real cfg1 operator:
    the matvec on the FP64 tensor pipe (h2b_mrhs.cu) timed with CUDA events, and a block
    GMRES(30) solve to 1e-6 of 64 seeded N(0,1) right-hand sides (host in, host out)."""
    if rank != 0:
        return None
    pk, ex = load(1)
    if pk is None:
        return None
    import ctypes as C
    import torch
    from paper_1703_01175_b200 import H2Operator, _abi, block_gmres_solve
    op = H2Operator(pk, device=local)
    L = _abi.lib()
    rng = np.random.default_rng(64)
    B = rng.standard_normal((pk.n, q)) + 1j * rng.standard_normal((pk.n, q))
    dev = torch.device(f"cuda:{local}")
    xd = torch.from_numpy(B[pk.perm]).to(dev)
    yd = torch.empty_like(xd)
    st = torch.cuda.current_stream(dev)

    def mv():
        _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), q,
                                     C.c_void_p(st.cuda_stream)))
    for _ in range(3):
        mv()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        mv()
    e1.record(st)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / 20
    nl = C.c_int64()
    _abi.check(L.h2b_query(op.handle, _abi.Q_MRHS_LAUNCHES, C.byref(nl)))
    block_gmres_solve(op, B, tol=1e-6, restart=30, max_iter=2)  # warm-up (cuSOLVER/cuBLAS handles)
    X, rep = block_gmres_solve(op, B, tol=1e-6, restart=30, max_iter=600)
    res = np.linalg.norm(op.matmat(X) - B, axis=0) / np.linalg.norm(B, axis=0)
    fp64_peak = 37.1e12  # measured DMMA/DFMA throughput, profiles/r01_fp64_peak.json
    out = {"config": f"cfg1 cube 16^3 (N=4096), q={q} seeded N(0,1) right-hand sides",
           "matvec_ms": ms, "value": pk.n * q / (ms * 1e-3), "unit": "unknowns*RHS/s",
           "tflops": pk.flops(q) / (ms * 1e-3) / 1e12,
           "frac_fp64_peak": pk.flops(q) / (ms * 1e-3) / fp64_peak,
           "kernel": "k_zgemm_grouped (DMMA m8n8k4, FP64 tensor pipe)", "launches": int(nl.value),
           "block_gmres": {"restart": 30, "tol": 1e-6, "iterations": rep.iterations,
                           "solve_s": rep.wall_time, "converged": rep.converged,
                           "max_true_rel_residual": float(res.max())}}
    op.close()
    return out


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    pk, ex = load(a.config)
    if pk is None:
        print(json.dumps({"impl": "reference", "unavailable": f"data/cfg{a.config}.npz missing"}))
        return 0
    x = ex["x"][:, 0]
    if pk.dbuf.size == 0:  # structure-exact operator: the CPU path needs the near-field on host
        from paper_1703_01175_b200.nearfield import assemble_near, geometry_arrays
        pk.dbuf = assemble_near(pk, *geometry_arrays(pk.meta["geometry"]))
    from oracle import h2_oracle as ho
    threads = os.cpu_count() or 1
    try:  # every host thread for the BLAS calls of the reference path
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=threads)
    except Exception:
        limiter, threads = None, 1
    for _ in range(max(1, a.warmup)):
        ho.matvec(pk, x)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        ho.matvec(pk, x)
    dt = (time.perf_counter() - t0) / a.steps
    if limiter is not None:
        limiter.restore_original_limits()
    v = pk.n / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic N(0,1) RHS (seed 0) on the reference-built operator",
            "config": config_desc(a.config, pk), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{a.steps} full matvecs of cfg{a.config} (oracle/h2_oracle.py "
                                       "restates arith.matvec loop-for-loop: a Python loop of small "
                                       f"numpy/OpenBLAS products, BLAS allowed {threads} threads)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_partitioned(a, pk, ex, rank, world, local, emit=True):
    """N GPUs, one process each: the operator is partitioned by subtree (SURVEY.md §8e,
    paper_1703_01175_b200/dist.py) — each rank owns a contiguous slice of rows and the
    matching bases / coupling rows / near-field rows; one NCCL all-gather of x and x̂ per
    matvec.  Total work is fixed (the whole operator), so scaling is "strong"."""
    import torch
    import torch.distributed as dist
    from paper_1703_01175_b200.dist import DistH2Operator
    from paper_1703_01175_b200.shard import PHASES
    from paper_1703_01175_b200.timing import L2Flusher
    dev = torch.device(f"cuda:{local}")
    op = DistH2Operator(pk, device=local, rank=rank, world=world, exchange=getattr(a, "exchange", "auto"))
    sl = slice(op.row0, op.row0 + op.nrows)
    xp_full = ex["x"][pk.perm, 0]
    xl = torch.from_numpy(xp_full[sl].copy()).to(dev)
    stream = torch.cuda.current_stream(dev)
    flush = L2Flusher(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    yl_buf = torch.empty_like(xl)
    for _ in range(max(3, a.warmup)):
        op.matvec_local(xl, out=yl_buf)
    barrier()
    with ClockSampler(local) as clk:
        time.sleep(0.25)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.steps)]
        for s, e in ev:
            flush.flush()
            if world > 1:
                dist.barrier()  # all ranks start the step together (the all-gather couples them)
            s.record(stream)
            y = op.matvec_local(xl, out=yl_buf)
            e.record(stream)
        barrier()
    ms = sum(s.elapsed_time(e) for s, e in ev) / a.steps
    # end to end: pinned host slice in, host slice out, every step
    xh = torch.from_numpy(xp_full[sl].copy()).pin_memory()
    t_e2e = []
    for _ in range(a.steps):
        barrier()
        t0 = time.perf_counter()
        yh = op.matvec_local(xh.to(dev, non_blocking=True)).cpu()
        t_e2e.append(time.perf_counter() - t0)
    e2e_s = float(np.median(t_e2e))  # wall clock per call: median (host jitter)
    exch_ms = op.exchange_ms(reps=10)
    ms, e2e_s, exch_ms = max_over_ranks([ms, e2e_s, exch_ms], dev)
    # parity: gather every rank's rows on rank 0
    yl = y.cpu().numpy()
    parts = [None] * world
    if world > 1:
        dist.all_gather_object(parts, (op.row0, yl))
    else:
        parts = [(op.row0, yl)]
    launches = sum(int(op.plan.phases[ph][0].size) for ph in PHASES)
    if rank == 0:
        yp = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
        relerr = (float(np.linalg.norm(yp - ex["y"][pk.perm, 0]) / np.linalg.norm(ex["y"][:, 0]))
                  if "y" in ex else None)
        peak, peak_src = peaks()
        alg = pk.algorithmic_bytes(1)
        line = {
            "metric": METRIC, "value": pk.n / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic: reference-built operator of BASELINE config, N(0,1) RHS (seed 0)",
            "config": config_desc(a.config, pk),
            "parallelism": f"subtree partition x{world} (level-log2(N) clusters); exchange of x and "
                           "x-hat per matvec: " + ("fused into the upward-pass kernels as NVLink P2P "
                                                   "stores + one barrier" if op.exchange_mode == "p2p"
                                                   else "one NCCL all-gather"),
            "l2": "flushed before every timed step",
            "roofline": {"bound": "hbm", "kernel": "whole partitioned matvec step (grouped GEMV "
                         "plan kernels per rank, max over ranks)", "achieved": alg / (ms * 1e-3) / 1e9,
                         "peak": peak * world, "unit": "GB/s",
                         "frac": alg / (ms * 1e-3) / 1e9 / (peak * world), "traffic": None,
                         "peak_source": peak_src + f" x {world} GPUs"},
            "e2e": {"value": pk.n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * pk.n,
                    "d2h_bytes_per_step": 16 * pk.n, "ms_per_call": e2e_s * 1e3},
            "gpu_launches": launches * a.steps, "gpu_launches_per_step": launches,
            "clocks": clk.summary(), "parity_relerr_vs_reference": relerr,
            "exchange_bytes_per_step": 16 * op.part.chunk * world,
            "exchange_ms": exch_ms,
            "exchange": op.exchange_mode,
        }
        if not emit:
            return line
        print(json.dumps(line))
    if not emit:
        return None
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_single(a, pk, ex, rank, world, local, steps=None, extras=True):
    """One GPU: the whole operator on this device, q = 1; L2 flushed before every timed step."""
    import ctypes as C
    import torch
    from paper_1703_01175_b200 import H2Operator, _abi, matvec as h2_matvec
    steps = steps or a.steps
    dev = torch.device(f"cuda:{local}")
    op = H2Operator(pk, device=local)
    L = _abi.lib()
    _abi.check(L.h2b_prepare_handle(op.handle), "prepare")
    x = torch.from_numpy(ex["x"][pk.perm, rank % ex["x"].shape[1]].copy()).to(dev)  # own RHS
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    from paper_1703_01175_b200.timing import L2Flusher
    flush = L2Flusher(dev)

    def mv():
        _abi.check(L.h2b_matvec_perm(op.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1, sh))

    def timed(fn, k, flush_l2=True):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for s, e in ev:
            if flush_l2:
                flush.flush()  # evict L2 (126 MB) before every timed step; not timed
            # a 20 us device spin before the start event: the host-side launch of the step
            # overlaps it, so the event pair brackets the device work (as in a solver loop,
            # where launches are queued ahead of the GPU)
            _abi.check(L.h2b_spin_ns(20000, sh))
            s.record(stream)
            fn()
            e.record(stream)
        torch.cuda.synchronize(dev)
        return sum(s.elapsed_time(e) for s, e in ev) / k  # ms

    for _ in range(max(3, a.warmup)):
        mv()
    # the warm-up steps proper are the timed step itself (L2 flush, spin, step), untimed: the first
    # flushed step of a process is a one-off (~80 us measured: first cold pass over the tables)
    timed(mv, max(3, a.warmup))
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        time.sleep(0.25)  # let the sampler start
        ms = timed(mv, steps)
        ms_warm = timed(mv, steps, flush_l2=False)
        # calibration: a plain cold read of as many bytes as the matvec's algorithmic traffic
        # through libh2b's TMA bulk-copy ring (h2b_stream_read: the near-field kernel's access
        # pattern without math), same flush and timing — the attainable streaming time at this
        # size (skipped when that buffer does not fit beside the operator: at such sizes the
        # cold read runs at the copy peak anyway)
        free_b, _ = torch.cuda.mem_get_info(dev)
        ms_read = None
        if pk.algorithmic_bytes(1) < 0.8 * free_b:
            nb = int(pk.algorithmic_bytes(1)) // 16 * 16
            cal = torch.ones(nb // 8, dtype=torch.float64, device=dev)
            sink = torch.zeros(1, dtype=torch.float64, device=dev)
            ms_read = timed(lambda: _abi.check(L.h2b_stream_read(C.c_void_p(cal.data_ptr()), nb,
                                                                 C.c_void_p(sink.data_ptr()), sh)),
                            max(5, min(steps, 10)))
            del cal
        for _ in range(3):  # keep the device busy for a few more clock samples
            timed(mv, steps)
    torch.cuda.synchronize(dev)
    ms, ms_warm = max_over_ranks([ms, ms_warm], dev)
    # parity guard on the measured output
    torch.cuda.synchronize(dev)
    yp = y.cpu().numpy()
    yy = np.empty_like(yp)
    yy[pk.perm] = yp
    relerr = (float(np.linalg.norm(yy - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0]))
              if "y" in ex else None)  # structure-exact operator: no reference output

    # the byte-dominant kernel alone: the same step with the far-field launch switched off
    # (H2B_OPT_DEBUG bit 1: timing only, y is then wrong and is not used)
    dominant = None
    mega_on = C.c_int64()
    _abi.check(L.h2b_query(op.handle, _abi.Q_MEGA, C.byref(mega_on)))
    if mega_on.value:
        _abi.check(L.h2b_set_option(op.handle, _abi.OPT_DEBUG, 2))
        for _ in range(3):
            mv()
        ms_near = max_over_ranks([timed(mv, steps)], dev)[0]
        _abi.check(L.h2b_set_option(op.handle, _abi.OPT_DEBUG, 0))
        nb = pk.near_bytes(1)
        dominant = {"kernel": "k_near_stream (near-field, alone: the step without its far-field launch)",
                    "alg_bytes_per_launch": nb, "ms_per_launch": ms_near,
                    "achieved": nb / (ms_near * 1e-3) / 1e9}

    # end to end through the reference-facing drop-in: matvec(h2, x) with a numpy (pageable)
    # x in, a fresh numpy y out (arith.py:108-117) — h2b_matvec_host stages the pageable buffers
    # through its own pinned ones; beside it the same C-ABI call on pinned caller buffers
    xn = ex["x"][:, 0].copy()
    for _ in range(3):
        h2_matvec(op, xn)
    t_e2e = []
    for _ in range(steps):
        t0 = time.perf_counter()
        yn = h2_matvec(op, xn)
        t_e2e.append(time.perf_counter() - t0)
    e2e_s = float(np.median(t_e2e))  # wall clock per call: median (host jitter)
    e2e_s = max_over_ranks([e2e_s], dev)[0]
    e2e_relerr = (float(np.linalg.norm(yn - ex["y"][:, 0]) / np.linalg.norm(ex["y"][:, 0]))
                  if "y" in ex else None)
    xh = torch.from_numpy(ex["x"][:, 0].copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()

    def e2e_call():
        _abi.check(L.h2b_matvec_host(op.handle, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1))

    for _ in range(3):
        e2e_call()
    t_pin = []
    for _ in range(steps):
        t0 = time.perf_counter()
        e2e_call()
        t_pin.append(time.perf_counter() - t0)
    e2e_pinned_s = float(np.median(t_pin))

    nlaunch, mega, tree_q = C.c_int64(), C.c_int64(), C.c_int64()
    _abi.check(L.h2b_query(op.handle, _abi.Q_LAUNCHES_Q1, C.byref(nlaunch)))
    _abi.check(L.h2b_query(op.handle, _abi.Q_TREE, C.byref(tree_q)))
    tree_on = tree_q.value != 0
    _abi.check(L.h2b_query(op.handle, _abi.Q_MEGA, C.byref(mega)))
    peak, peak_src = peaks()
    alg_bytes = pk.algorithmic_bytes(1)
    achieved = alg_bytes / (ms * 1e-3) / 1e9
    # DRAM bytes per step (read + write of both kernels) from the committed ncu launch list of
    # this configuration and far-field variant (profiles/step_traffic.json)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "step_traffic.json")
    if os.path.exists(prof):
        try:
            ent = json.load(open(prof)).get(f"cfg{a.config}", {}).get("tree" if tree_on else "mega")
            traffic = ent["bytes"] if ent else None
        except Exception:
            traffic = None
    unknowns = pk.n * 1
    line = {
        "metric": METRIC,
        "value": world * unknowns / (ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": steps,
        "warmup": a.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "complex128 (f64)",
        "data": "synthetic: reference-built operator of BASELINE config, N(0,1) RHS (seed 0)",
        "config": config_desc(a.config, pk),
        "l2": "flushed before every timed step (256 MiB write + 256 MiB read: clean L2)",
        "parallelism": "1 GPU (the whole operator)",
        "achieved_gbs_total": pk.algorithmic_bytes(1) / (ms * 1e-3) / 1e9,
        "hbm_frac_total": pk.algorithmic_bytes(1) / (ms * 1e-3) / 1e9 / peak,
        "roofline": {"bound": "hbm",
                     "kernel": ("whole matvec step: k_near_stream (near-field, ~83% of B_alg) "
                                "concurrent with " + ("k_far_tree (far field as subtree programs)"
                                                      if tree_on else "k_mega (far-field task graph)") +
                                "; B_alg = 16(E_V+E_T+E_S+E_D) + 32(N+K) bytes per step"
                                if int(nlaunch.value) == 2 and int(mega.value) else
                                f"whole matvec step ({int(nlaunch.value)} launches); B_alg = "
                                "16(E_V+E_T+E_S+E_D) + 32(N+K) bytes per step"),
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "ms_per_launch": ms,
                     "alg_bytes_per_launch": alg_bytes,
                     "warm_l2_ms_per_launch": ms_warm,
                     "warm_l2_achieved": alg_bytes / (ms_warm * 1e-3) / 1e9,
                     "cold_read_same_bytes_ms": ms_read,
                     "frac_of_cold_read": ms_read / ms if ms_read else None},
        "dominant_kernel": (dict(dominant, peak=peaks()[0], unit="GB/s",
                                 frac=dominant["achieved"] / peaks()[0]) if dominant else None),
        "e2e": {"value": world * unknowns / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * pk.n,
                "d2h_bytes_per_step": 16 * pk.n, "ms_per_call": e2e_s * 1e3,
                "call": "paper_1703_01175_b200.matvec(h2, x): numpy x in, fresh numpy y out",
                "parity_relerr_vs_reference": e2e_relerr},
        "e2e_pinned": {"value": world * unknowns / e2e_pinned_s, "unit": UNIT,
                       "ms_per_call": e2e_pinned_s * 1e3,
                       "call": "h2b_matvec_host on pinned caller buffers (one CUDA graph per call)"},
        "gpu_launches": int(nlaunch.value) * steps,
        "gpu_launches_per_step": int(nlaunch.value),
        "clocks": clk.summary(),
        "parity_relerr_vs_reference": relerr,
    }
    op.close()
    return line


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import ctypes as C
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        backend = os.environ.get("H2B_BENCH_BACKEND", "nccl")  # gloo: functional tests only
        # NCCL's init log (one line per rank and channel setup) on stderr: the rank count and the
        # NVLink / NVLS transport are visible in the run's log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    from paper_1703_01175_b200 import H2Operator, _abi

    pk, ex = load(a.config)
    if pk is None:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "error": f"data/cfg{a.config}.npz missing"}))
        return 1
    if world > 1 or a.partitioned:
        # N GPUs: the operator partitioned by subtree: strong scaling of one RHS
        line = run_partitioned(a, pk, ex, rank, world, local, emit=False)
        if rank == 0 and line is None:
            return 1
    else:
        line = run_single(a, pk, ex, rank, world, local)
    if world == 1:
        gm = gmres_bench(rank, world, local) if not a.no_gmres else None
        if gm:
            line["gmres"] = gm
        bc = bicgstab_bench(rank, local) if not a.no_gmres else None
        if bc:
            line["bicgstab"] = bc
        mr = mrhs_bench(rank, local) if not a.no_gmres else None
        if mr:
            line["multi_rhs"] = mr
        if rank == 0 and not a.no_cpu_baseline:
            t_cpu, n_cpu = cpu_port_time(pk, ex["x"][:, 0], a.cpu_seconds)
            line["cpu_baseline"] = {"value": pk.n / t_cpu, "unit": UNIT, "cores": 1, "kind": "port",
                                    "sample": f"{n_cpu} full cfg{a.config} matvecs in {t_cpu * n_cpu:.1f} s "
                                              "(oracle/h2_oracle.py restates arith.matvec loop-for-loop)",
                                    "cpu": os.cpu_count()}
    # BASELINE's scaling config at every N: the 2M-unknown cube (cfg4, structure-exact: the
    # reference block structure and ranks, payloads generated on each device) — one GPU holds the
    # whole 140 GB operator at N = 1, N > 1 partitions it by subtree (strong scaling of one RHS).
    # A failure here must not cost the headline line.
    cube_k = int(os.environ.get("H2B_BENCH_CUBE_CONFIG", "4"))  # another config: functional tests
    if not a.no_cube and a.config != cube_k:
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        cube, errs = None, []
        try:
            pk4, ex4 = load(cube_k)
            if pk4 is None:
                raise FileNotFoundError(f"fixtures/cfg{cube_k}_structure.npz")
            sub = argparse.Namespace(**dict(vars(a), config=cube_k, steps=min(a.steps, 5), warmup=3,
                                            exchange="auto"))
            if world > 1:
                cube = run_partitioned(sub, pk4, ex4, rank, world, local, emit=False)
            else:
                cube = run_single(sub, pk4, ex4, rank, world, local, steps=sub.steps)
        except Exception as e:  # noqa: BLE001
            errs.append(f"{type(e).__name__}: {e}"[:300])
        if rank == 0:
            line["cube_strong"] = (
                {"error": errs} if cube is None else
                dict({k: cube[k] for k in ("value", "unit", "ms_per_step", "scaling", "roofline", "e2e",
                                           "gpu_launches_per_step", "parallelism", "n_gpus")
                      if k in cube},
                     config=cube["config"],
                     **{k: cube[k] for k in ("exchange_bytes_per_step", "exchange_ms", "exchange")
                        if k in cube}))
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
