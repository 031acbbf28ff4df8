"""Per-rank device programs of the G-way subtree partition, timed one at a time on ONE B200.

Every rank's plan (shard.plan_shard, payloads generated on the device: seeded far field,
near-field sampled from the geometry) runs its whole q = 1 step — UP_OWN, UP_TOP, COUPLE,
DOWN, NEAR — as one CUDA graph with the exchange buffer already holding every rank's x slice
and x̂ rows (the state right after the exchange), L2 flushed before every timed step.  A rank's
device time does not depend on the other GPUs, so max over ranks is the compute part of a
G-GPU step; the exchange (x and own x̂ to every peer, `exchange_bytes` per rank) is not
measured here.  Optional parity (--check): the ranks' outputs, stitched, against the
single-GPU structure-exact operator (only when both fit one GPU).

usage: rank_programs.py STRUCTURE.npz G [--ranks 0,3] [--reps 10] [--check]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("structure")
    ap.add_argument("G", type=int)
    ap.add_argument("--ranks", default="")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--phases", action="store_true", help="also time each phase (events between launches)")
    ap.add_argument("--sequential", action="store_true", help="phases one after another (no concurrent near-field)")
    a = ap.parse_args()
    from paper_1703_01175_b200.dist import CudaPlanEngine
    from paper_1703_01175_b200.pack import load_packed
    from paper_1703_01175_b200.shard import (PH_COUPLE, PH_DOWN, PH_NEAR, PH_UP_OWN, PH_UP_TOP,
                                             partition, plan_shard)
    from paper_1703_01175_b200.timing import L2Flusher
    pk = load_packed(a.structure, near_on_host=False, far_on_host=False)
    G = a.G
    part = partition(pk, G)
    ranks = [int(r) for r in a.ranks.split(",")] if a.ranks else list(range(G))
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal(pk.n) + 1j * rng.standard_normal(pk.n)).to(dev)
    flush = L2Flusher("cuda")
    ch = part.chunk
    out, Y = [], (torch.empty(pk.n, dtype=torch.complex128, device=dev) if a.check else None)

    def x_buffer():
        xb = torch.zeros((part.xlen, 1), dtype=torch.complex128, device=dev)
        for r in range(G):  # every rank's x slice (the post-exchange state)
            r0, r1 = int(part.row0[r]), int(part.row0[r]) + int(part.nrows[r])
            xb[r * ch:r * ch + (r1 - r0), 0] = x[r0:r1]
        return xb

    exchanged = None
    if a.check:  # pass 1: every rank's own x̂ rows, so pass 2 sees the true exchanged buffer
        exchanged = x_buffer()
        for g in range(G):
            p = plan_shard(pk, G, g, part, device_payloads=True)
            eng = CudaPlanEngine(p, 0)
            xb = x_buffer()
            eng.run(PH_UP_OWN, xb, torch.zeros_like(xb), torch.zeros((p.nrows, 1), dtype=torch.complex128, device=dev), 1)
            exchanged[g * ch:(g + 1) * ch] = xb[g * ch:(g + 1) * ch]
            eng.close()
            del eng
            torch.cuda.empty_cache()
    for g in ranks:
        t0 = time.time()
        p = plan_shard(pk, G, g, part, device_payloads=True)
        t_plan = time.time() - t0
        t0 = time.time()
        eng = CudaPlanEngine(p, 0)
        torch.cuda.synchronize()
        t_fill = time.time() - t0
        xb = x_buffer() if exchanged is None else exchanged.clone()
        xh = torch.zeros_like(xb)
        y = torch.zeros((p.nrows, 1), dtype=torch.complex128, device=dev)
        st = torch.cuda.Stream(dev)
        st.wait_stream(torch.cuda.current_stream())

        def step():  # as DistH2Operator._body after the exchange
            eng.run(PH_UP_OWN, xb, xh, y, 1)
            if a.sequential:
                for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
                    eng.run(ph, xb, xh, y, 1)
            else:
                eng.run_tail(xb, xh, y, 1)

        with torch.cuda.stream(st):
            step()  # warm (lazy preparation outside the capture)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                step()
        torch.cuda.synchronize()
        times = []
        for _ in range(a.reps):
            flush.flush()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            gr.replay()
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        ms = float(np.median(times))
        phase_ms = None
        if a.phases:  # per phase, outside the graph (launch overheads included), L2 flushed per step
            names = ("UP_OWN", "UP_TOP", "COUPLE", "DOWN", "NEAR")
            acc = np.zeros(5)
            for _ in range(a.reps):
                flush.flush()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
                ev[0].record()
                for i, ph in enumerate((PH_UP_OWN, PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR)):
                    eng.run(ph, xb, xh, y, 1)
                    ev[i + 1].record()
                torch.cuda.synchronize()
                acc += [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
            phase_ms = dict(zip(names, (acc / a.reps).round(4).tolist()))
        rec = {"rank": g, "G": G, "rows": int(p.nrows), "ms": ms, "payload_bytes": p.payload_bytes(),
               "payload_gbs": p.payload_bytes() / (ms * 1e-3) / 1e9, "plan_s": round(t_plan, 2),
               "fill_s": round(t_fill, 2), "phase_ms": phase_ms}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        if a.check:
            Y[p.row0:p.row0 + p.nrows] = y[:, 0]
        del gr
        eng.close()
        del eng, xb, xh, y
        torch.cuda.empty_cache()
    worst = max(out, key=lambda r: r["ms"])
    B = pk.algorithmic_bytes()
    summary = {"structure": os.path.basename(a.structure), "n": pk.n, "G": G, "ranks_timed": len(out),
               "max_rank_ms": worst["ms"], "slowest_rank": worst["rank"],
               "algorithmic_bytes": B,
               "projected_unknowns_per_s": pk.n / (worst["ms"] * 1e-3) if len(out) == G else None,
               "projected_alg_gbs": B / (worst["ms"] * 1e-3) / 1e9 if len(out) == G else None,
               "exchange_bytes_per_rank": 16 * ch * G,
               "note": "compute part only (each rank's program alone on one B200); the exchange is not measured"}
    if a.check and len(out) == G:
        from paper_1703_01175_b200 import H2Operator
        op = H2Operator(pk)
        ref = torch.empty_like(Y)
        op.matvec_perm(x, out=ref)
        summary["relerr_vs_single_gpu"] = float(torch.linalg.norm(Y - ref) / torch.linalg.norm(ref))
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
