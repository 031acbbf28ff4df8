"""Multi-GPU H² matvec and GMRES: subtree partition + one all-gather per matvec.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank g
holds the shard of `shard.plan_shard` (its subtree's bases, coupling rows and
near-field rows) in a libh2b plan handle and the Krylov vectors' slice
``[row0_g, row0_g + nrows_g)`` of the permuted index space.  Per matvec the
only communication is ONE ``all_gather_into_tensor`` of the exchange buffer
(each rank's x slice and its own x̂ values, SURVEY.md §8e (i)+(ii) fused into a
single collective); per Arnoldi step of GMRES the dots and norms are
``all_reduce`` sums of per-rank partials.

The compute engine is pluggable so the host logic (partition, exchange
layout, collectives, GMRES) is exercised unchanged by the CPU tests on gloo:
`CudaPlanEngine` (the product: libh2b ``h2b_plan_run`` on the rank's GPU) or
a test engine that interprets the same plan on the CPU.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _abi
from .krylov import SolveReport
from .shard import (N_PAY, PH_COUPLE, PH_DOWN, PH_LEAFBACK, PH_NEAR, PH_UP_OWN, PH_UP_TOP, PHASES,
                    partition, plan_shard)

_UPLOAD_CHUNK = 1 << 30


class CudaPlanEngine:
    """A shard plan resident on one B200 (libh2b plan handle)."""

    def __init__(self, plan, device):
        L = _abi.lib()
        self.device = int(device)
        sizes = plan.payload_sizes() if hasattr(plan, "payload_sizes") else [int(a.size) for a in plan.payloads]
        elems = (C.c_int64 * N_PAY)(*sizes)
        h = C.c_void_p()
        _abi.check(L.h2b_plan_create(self.device, N_PAY, elems, C.byref(h)), "h2b_plan_create")
        self.handle = h
        for i, a in enumerate(plan.payloads):
            b = np.ascontiguousarray(a).view(np.uint8)
            for off in range(0, b.size, _UPLOAD_CHUNK):
                ch = b[off:off + _UPLOAD_CHUNK]
                _abi.check(L.h2b_plan_upload(h, i, ch.ctypes.data, ch.size, off), "h2b_plan_upload")
        fills = getattr(plan, "fills", None)
        if fills is not None:  # structure-exact payloads generated on this device
            from .synthetic import SCALES
            for i, d in enumerate(fills["synth"]):
                if d.size:
                    d = np.ascontiguousarray(d)
                    sec = int(d[0, 5])
                    _abi.check(L.h2b_plan_fill_synthetic(h, i, d.ctypes.data, int(d.shape[0]),
                                                         int(fills["seed"]), SCALES[sec]),
                               "h2b_plan_fill_synthetic")
            if fills["near"].size:
                from .nearfield import geometry_arrays, self_term
                centers, chi, k0, vol = geometry_arrays(fills["geometry"])
                diag = k0 ** 2 * self_term(vol, k0)
                d = np.ascontiguousarray(fills["near"])
                perm = np.ascontiguousarray(fills["perm"], dtype=np.int64)
                centers = np.ascontiguousarray(centers, dtype=np.float64)
                chi = np.ascontiguousarray(chi, dtype=np.complex128)
                _abi.check(L.h2b_plan_fill_near(h, 4, d.ctypes.data, int(d.shape[0]), perm.ctypes.data,
                                                int(perm.size), centers.ctypes.data, chi.ctypes.data,
                                                float(k0), float(vol), float(diag.real), float(diag.imag)),
                           "h2b_plan_fill_near")
        g = np.ascontiguousarray(getattr(plan, "gather", np.zeros(0, np.int32)), dtype=np.int32)
        _abi.check(L.h2b_plan_set_gather(h, g.ctypes.data_as(C.POINTER(C.c_int32)), int(g.size)),
                   "h2b_plan_set_gather")
        for ph in sorted(plan.phases):
            counts, items, segs = plan.phases[ph]
            _abi.check(L.h2b_plan_set_phase(h, ph, int(counts.size),
                                            counts.ctypes.data_as(C.POINTER(C.c_int64)),
                                            items.ctypes.data, int(items.size), segs.ctypes.data,
                                            int(segs.size)), "h2b_plan_set_phase")
        cf = getattr(plan, "couple_fast", None)
        if cf is not None and cf["items"].size:  # q = 1 coupling on the panel kernels
            _abi.check(L.h2b_plan_set_couple_fast(h, cf["items"].ctypes.data, int(cf["items"].size),
                                                  cf["xcol"].ctypes.data_as(C.POINTER(C.c_int32)),
                                                  int(cf["xcol"].size)), "h2b_plan_set_couple_fast")
        nf = getattr(plan, "near_fast", None)
        self.has_near_fast = bool(nf is not None and nf["items"].size)
        self._side = self._ev = None
        if self.has_near_fast:  # q = 1 near-field on the streaming kernel
            _abi.check(L.h2b_plan_set_near_fast(h, nf["items"].ctypes.data, int(nf["items"].size),
                                                nf["blks"].ctypes.data, int(nf["blks"].size),
                                                int(nf["ns"]), int(nf["R"])), "h2b_plan_set_near_fast")

    def set_peers(self, ptrs):
        arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        _abi.check(_abi.lib().h2b_plan_set_peers(self.handle, arr, len(ptrs)), "h2b_plan_set_peers")

    def bcast_rows(self, buf, row0, nrows, q, stream=None):
        torch = __import__("torch")
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        _abi.check(_abi.lib().h2b_plan_bcast_rows(self.handle, C.c_void_p(buf.data_ptr()), int(row0),
                                                  int(nrows), int(q), C.c_void_p(st.cuda_stream)),
                   "h2b_plan_bcast_rows")

    def run(self, phase, xbuf, yhat, y, q, stream=None):
        torch = __import__("torch")
        st = torch.cuda.current_stream(self.device) if stream is None else stream  # (capturing)
        _abi.check(_abi.lib().h2b_plan_run(self.handle, phase, C.c_void_p(xbuf.data_ptr()),
                                           C.c_void_p(xbuf.data_ptr()), C.c_void_p(yhat.data_ptr()),
                                           C.c_void_p(y.data_ptr()), int(q),
                                           C.c_void_p(st.cuda_stream)), "h2b_plan_run")

    def run_tail(self, xbuf, yhat, y, q):
        """The phases after the exchange: UP_TOP → COUPLE → DOWN (the far field), and NEAR.  At
        q = 1 with the streaming near-field, the near-field (it reads only x) runs on a second
        stream beside the latency-bound far-field chain, and the leaf back-transform (it needs
        both) after the join — capturable into the caller's CUDA graph."""
        torch = __import__("torch")
        if not (q == 1 and self.has_near_fast):
            for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
                self.run(ph, xbuf, yhat, y, q)
            return
        main = torch.cuda.current_stream(self.device)
        if self._side is None:  # high priority: the chain's CTAs go ahead of the near-field's
            self._side = torch.cuda.Stream(self.device, priority=-1)
            self._ev = (torch.cuda.Event(), torch.cuda.Event())
        fork, join = self._ev
        fork.record(main)
        self._side.wait_event(fork)
        for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN):
            self.run(ph, xbuf, yhat, y, 1, stream=self._side)
        self.run(_abi.PLAN_PHASE_NEAR_FAST, xbuf, yhat, y, 1, stream=main)
        join.record(self._side)
        main.wait_event(join)
        self.run(PH_LEAFBACK, xbuf, yhat, y, 1, stream=main)

    def device_bytes(self):
        return int(_abi.lib().h2b_plan_device_bytes(self.handle))

    def close(self):
        if self.handle:
            _abi.lib().h2b_plan_destroy(self.handle)
            self.handle = None


class DistH2Operator:
    """Rank-local view of the subtree-partitioned operator.

    ``matvec_local(x_local)`` takes this rank's rows of x (permuted order,
    (nrows,) or (nrows, q) complex128 torch tensor on the rank's device) and
    returns its rows of y = S x.  Collective: every rank must call it.
    """

    def __init__(self, pk, group=None, device=None, engine=None, rank=None, world=None,
                 exchange="auto"):
        """``engine``: None (libh2b on ``device`` / the current CUDA device) or a factory
        ``plan -> engine`` (the CPU tests pass the plan interpreter).

        ``exchange``: "p2p" — the x̂ all-gather fused into the UP_OWN kernels, which store into
        every rank's exchange buffer over NVLink (CUDA IPC mappings), then one barrier collective;
        "allgather" — one NCCL all-gather of the exchange buffer; "auto" — p2p when every pair
        of GPUs has peer access under NCCL, else allgather."""
        import torch
        import torch.distributed as dist
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rank, self.world = int(rank), int(world)
        self.part = partition(pk, self.world)
        backend = dist.get_backend(group) if (dist.is_initialized() and self.world > 1) else "nccl"
        want_p2p = (exchange in ("auto", "p2p") and engine is None and self.world > 1
                    and backend == "nccl")
        if want_p2p and exchange == "auto":
            want_p2p = _peer_access_everywhere(group, torch.cuda.current_device() if device is None
                                               else int(device), self.world)
        self.exchange_mode = "p2p" if want_p2p else "allgather"
        self.plan = plan_shard(pk, self.world, self.rank, self.part, bcast=want_p2p,
                               device_payloads=engine is None)
        self.n = int(pk.n)
        self.row0, self.nrows = self.plan.row0, self.plan.nrows
        if engine is None:
            dev = torch.cuda.current_device() if device is None else device
            engine = CudaPlanEngine(self.plan, dev)
            self.device = torch.device(f"cuda:{engine.device}")
        else:
            engine = engine(self.plan)
            self.device = torch.device(getattr(engine, "device_name", "cpu"))
        self.engine = engine
        self._ws = {}
        self._graphs = {}
        backend = dist.get_backend(group) if (dist.is_initialized() and self.world > 1) else "nccl"
        self._host_staged = backend == "gloo" and self.device.type == "cuda"
        self._graph_ok = self.device.type == "cuda" and (self.world == 1 or backend == "nccl")
        self._slot = 0
        self._p2p = {}  # q -> (raw allocation, two exchange-buffer views, opened peer pointers)

    def _work(self, q):
        import torch
        if q not in self._ws:
            z = lambda r: torch.zeros((r, q), dtype=torch.complex128, device=self.device)  # noqa: E731
            xb = self._p2p_buffers(q)[self._slot] if self.exchange_mode == "p2p" else z(self.part.xlen)
            self._ws[q] = (xb, z(self.part.xlen), z(self.nrows), z(self.part.chunk))
        ws = self._ws[q]
        if self.exchange_mode == "p2p":  # alternate exchange buffers between matvecs
            ws = (self._p2p_buffers(q)[self._slot],) + ws[1:]
        return ws

    def _p2p_buffers(self, q):
        """Two exchange buffers in one IPC-shared allocation; peers mapped once per q."""
        if q not in self._p2p:
            import torch
            import torch.distributed as dist
            L = _abi.lib()
            elems = self.part.xlen * q
            raw = C.c_void_p()
            _abi.check(L.h2b_device_alloc(int(self.device.index), 32 * elems, C.byref(raw)),
                       "h2b_device_alloc")
            hd = (C.c_char * 64)()
            _abi.check(L.h2b_ipc_get_handle(raw, hd), "h2b_ipc_get_handle")
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(hd), group=self.group)
            peers = []
            for r in range(self.world):
                if r == self.rank:
                    continue
                ptr = C.c_void_p()
                buf = (C.c_char * 64).from_buffer_copy(handles[r])
                _abi.check(L.h2b_ipc_open(buf, C.byref(ptr)), "h2b_ipc_open")
                peers.append(ptr.value)
            self.engine.set_peers(peers)
            views = [_device_view(raw.value + 16 * elems * b, (self.part.xlen, q), self.device)
                     for b in range(2)]
            self._p2p[q] = (raw, views, peers)
        return self._p2p[q][1]

    def exchange(self, xbuf, send, q):
        """All-gather of every rank's chunk (x slice + own x̂) into the exchange buffer."""
        import torch
        import torch.distributed as dist
        ch = self.part.chunk
        g = self.rank
        if self.world == 1:
            return
        send.copy_(xbuf[g * ch:(g + 1) * ch])
        if self._host_staged:  # gloo with device buffers (functional tests): stage on the host
            out = torch.empty((self.world * ch,) + tuple(send.shape[1:]), dtype=send.dtype)
            dist.all_gather_into_tensor(torch.view_as_real(out), torch.view_as_real(send.cpu()),
                                        group=self.group)
            xbuf[:self.world * ch].copy_(out)
            return
        dist.all_gather_into_tensor(torch.view_as_real(xbuf[:self.world * ch]),
                                    torch.view_as_real(send), group=self.group)

    def allreduce_(self, t):
        """In-place sum over ranks of a real tensor (host-staged under gloo with CUDA tensors)."""
        import torch.distributed as dist
        if self.world == 1:
            return t
        if self._host_staged:
            c = t.cpu()
            dist.all_reduce(c, group=self.group)
            t.copy_(c)
        else:
            dist.all_reduce(t, group=self.group)
        return t

    def _body(self, q):
        """The matvec on the workspace of q columns: x slice already in the exchange buffer."""
        xbuf, yhat, y, send = self._work(q)
        if self.exchange_mode == "p2p":
            # fused exchange: x rows pushed to every peer, x̂ stored to every peer by the UP_OWN
            # epilogues; one barrier collective orders the peers' next phase after the stores
            _abi.check(_abi.lib().h2b_plan_set_peer_offset(self.engine.handle,
                                                           self._slot * self.part.xlen * q),
                       "h2b_plan_set_peer_offset")
            self.engine.bcast_rows(xbuf, self.rank * self.part.chunk, self.nrows, q)
            self.engine.run(PH_UP_OWN, xbuf, yhat, y, q)
            self._barrier()
        else:
            self.engine.run(PH_UP_OWN, xbuf, yhat, y, q)
            self.exchange(xbuf, send, q)
        tail = getattr(self.engine, "run_tail", None)  # the CPU plan interpreter has none
        if tail is not None:
            tail(xbuf, yhat, y, q)
        else:
            for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
                self.engine.run(ph, xbuf, yhat, y, q)

    def exchange_ms(self, reps=10, q=1):
        """Device time (ms, CUDA events, mean of ``reps``) of this rank's exchange step alone: the
        NCCL all-gather of the exchange buffer, or (p2p) the x-slice broadcast over NVLink plus the
        barrier collective — the x̂ stores of the p2p mode are fused into the upward-pass kernels
        and are not separable.  Collective: every rank must call it."""
        import torch
        xbuf, yhat, y, send = self._work(q)
        if self.world == 1 or self.device.type != "cuda":
            return 0.0

        def step():
            if self.exchange_mode == "p2p":
                self.engine.bcast_rows(xbuf, self.rank * self.part.chunk, self.nrows, q)
                self._barrier()
            else:
                self.exchange(xbuf, send, q)
        step()
        torch.cuda.synchronize(self.device)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            step()
        e.record()
        torch.cuda.synchronize(self.device)
        return s.elapsed_time(e) / reps

    def matvec_local(self, x_local, graph=True, out=None):
        """This rank's rows of S x.  On CUDA the whole step — the plan launches of every phase
        and the NCCL all-gather — is captured once per q into a CUDA graph and replayed.
        ``out``: a caller-owned (nrows,) / (nrows, q) tensor to write into (no allocation)."""
        import torch
        squeeze = x_local.dim() == 1
        xl = x_local.reshape(self.nrows, -1)
        q = xl.shape[1]
        xbuf, yhat, y, send = self._work(q)
        g, ch = self.rank, self.part.chunk
        xbuf[g * ch:g * ch + self.nrows].copy_(xl)
        if graph and self._graph_ok:
            key = (q, self._slot)
            cg = self._graphs.get(key)
            if cg is None:
                self._body(q)  # warm-up outside capture (NCCL communicator, attributes)
                torch.cuda.synchronize(self.device)
                cg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cg):
                    self._body(q)
                self._graphs[key] = cg
                xbuf[g * ch:g * ch + self.nrows].copy_(xl)
            cg.replay()
        else:
            self._body(q)
        if out is None:
            out = y.clone()
            res = out[:, 0] if squeeze else out
        else:
            out.reshape(self.nrows, -1).copy_(y)
            res = out
        if self.exchange_mode == "p2p":
            self._slot ^= 1
        return res

    def close(self):
        """Release the device resources: IPC mappings, exchange allocations, the plan handle."""
        L = _abi.lib()
        for raw, _views, peers in self._p2p.values():
            for ptr in peers:
                L.h2b_ipc_close(C.c_void_p(ptr))
            L.h2b_device_free(raw)
        self._p2p.clear()
        self._graphs.clear()
        self._ws.clear()
        if hasattr(self.engine, "close"):
            self.engine.close()

    def _barrier(self):
        """Stream-ordered barrier collective (NCCL all-reduce of one element)."""
        import torch
        import torch.distributed as dist
        if not hasattr(self, "_bar"):
            self._bar = torch.zeros(1, dtype=torch.float32, device=self.device)
        dist.all_reduce(self._bar, group=self.group)

    # ---- Krylov helper: global 2-norm over the row slices -------------------------
    def norm(self, a):
        """||a|| over all ranks: the rank's partial (libh2b reduction on CUDA), one all-reduce."""
        import torch
        if a.is_cuda:
            a = a.contiguous()
            s = torch.empty(1, dtype=torch.complex128, device=a.device)
            _abi.check(_abi.lib().h2b_zdotc_multi(C.c_void_p(a.data_ptr()), a.numel(), 1,
                                                  C.c_void_p(a.data_ptr()), a.numel(),
                                                  C.c_void_p(s.data_ptr()),
                                                  C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)),
                       "h2b_zdotc_multi")
            s = s.real.clone()
        else:
            s = (a.real * a.real + a.imag * a.imag).sum().reshape(1)
        self.allreduce_(s)
        return float(torch.sqrt(s)[0])


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can view a raw libh2b allocation."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape) + (2,), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _device_view(ptr, shape, device):
    import torch
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaArray(ptr, shape), device=device)
    return torch.view_as_complex(t)


def _peer_access_everywhere(group, dev, world):
    """True when this rank's GPU can store to every other rank's GPU (NVLink / NVSwitch)."""
    import torch
    import torch.distributed as dist
    devs = [None] * world
    props = torch.cuda.get_device_properties(dev)
    dist.all_gather_object(devs, (str(getattr(props, "uuid", dev)), dev), group=group)
    if len({d[0] for d in devs}) < world:
        return False  # two ranks on one GPU: no IPC peer mapping
    ok = all(torch.cuda.can_device_access_peer(dev, d[1]) for d in devs if d[1] != dev)
    flags = [None] * world
    dist.all_gather_object(flags, bool(ok), group=group)
    return all(flags)


def _givens(a, b):
    if b == 0.0:
        return 1.0, 0.0 + 0.0j, a
    if a == 0:
        return 0.0, 1.0 + 0.0j, complex(b)
    t = np.hypot(abs(a), b)
    ph = a / abs(a)
    return abs(a) / t, ph * b / t, ph * t


def dist_gmres_solve(op: DistH2Operator, b_local, tol=1e-6, restart=30, max_iter=1000):
    """Restarted GMRES(m), CGS2 Arnoldi, x0 = 0, on row-distributed vectors (collective).

    Same recurrence and stopping rule as the single-GPU ``gmres_solve`` (h2b_krylov.cu:
    h2b_gmres) and the CPU restatement (oracle/krylov_oracle.py::gmres_solve).  Each rank keeps
    its rows of the Arnoldi basis in device memory; one step is the partitioned matvec, two CGS
    passes (libh2b multi-dot → ONE all-reduce of the j+1 coefficients per pass → basis update,
    the second fused with ||w||^2 → one all-reduce), the device Givens recurrence
    (h2b_gmres_givens, which writes the step's residual into mapped pinned memory) and the
    normalisation by a device scalar.  Nothing is read back per step: the host checks the
    residual of step j while step j+1 is already queued, and syncs only at the end of a cycle
    (back substitution).  With the CPU plan interpreter (tests) the same recurrence runs on
    torch CPU tensors.
    """
    import torch
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be >= 1")
    if restart > 63:
        raise ValueError("restart must be <= 63")
    if op.device.type != "cuda":
        return _dist_gmres_host(op, b_local, tol, restart, max_iter)
    t0 = time.perf_counter()
    L = _abi.lib()
    dev = op.device
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    b = b_local.to(dev, torch.complex128).contiguous()
    bnrm = op.norm(b)
    if bnrm == 0.0:
        return torch.zeros_like(b), SolveReport(0, [], True, time.perf_counter() - t0)
    m, n = int(restart), op.nrows
    x = torch.zeros_like(b)
    r = b.clone()
    V = torch.zeros((m + 1, n), dtype=torch.complex128, device=dev)
    hv = torch.zeros(256, dtype=torch.complex128, device=dev)       # CGS coefficients, ||w||^2
    st = torch.zeros(int(L.h2b_gmres_state_elems(m)), dtype=torch.complex128, device=dev)
    o_g = (m + 1) * m
    o_scale = o_g + (m + 1) + 3 * m
    st[o_scale + 1] = bnrm                                           # {||b||, 0}
    # mapped pinned records written by the Givens kernel: {res_j, 0}, {hn_j, 0} per step j
    host_res = torch.zeros(4 * m, dtype=torch.float64).pin_memory()
    tmp = torch.empty_like(b)

    def ptr(t, off=0):
        return C.c_void_p(t.data_ptr() + 16 * off)

    def allreduce(t):
        if op.world > 1:
            op.allreduce_(torch.view_as_real(t))

    def step(j):
        w = V[j + 1]
        op.matvec_local(V[j], out=w)
        _abi.check(L.h2b_zdotc_multi(ptr(V), n, j + 1, ptr(w), n, ptr(hv), sh), "h2b_zdotc_multi")
        allreduce(hv[:j + 1])
        _abi.check(L.h2b_zgemv_sub(ptr(V), n, j + 1, ptr(hv), ptr(w), n, None, sh), "h2b_zgemv_sub")
        _abi.check(L.h2b_zdotc_multi(ptr(V), n, j + 1, ptr(w), n, ptr(hv, 64), sh), "h2b_zdotc_multi")
        allreduce(hv[64:65 + j])
        _abi.check(L.h2b_zgemv_sub(ptr(V), n, j + 1, ptr(hv, 64), ptr(w), n, ptr(hv, 128), sh),
                   "h2b_zgemv_sub")
        allreduce(hv[128:129])
        _abi.check(L.h2b_gmres_givens(ptr(st), m, j, ptr(hv), C.c_void_p(host_res.data_ptr()), sh),
                   "h2b_gmres_givens")
        _abi.check(L.h2b_zscale_dev(ptr(w), n, ptr(st, o_scale), sh), "h2b_zscale_dev")
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    it, history, converged = 0, [], False
    beta = bnrm
    while it < max_iter:
        if it > 0:
            beta = op.norm(r)
        st[o_g:o_g + m + 1] = 0
        st[o_g] = beta
        _abi.check(L.h2b_zaxpby(n, 1.0 / beta, 0.0, ptr(r), 0.0, 0.0, ptr(V[0]), sh), "h2b_zaxpby")
        # step j+1 is queued before the host reads step j's residual (h2b_gmres's scheme: a
        # speculative step writes only V[j+2], column j+1 of H and g[j+1..j+2], none of which the
        # back substitution of a cycle ending at j reads)
        it0, j_done = it, 0
        evs = [step(0)]
        for j in range(m):
            if j + 1 < m and it0 + j + 1 < max_iter:
                evs.append(step(j + 1))
            evs[j].synchronize()
            it += 1
            res, hn = float(host_res[4 * j]), float(host_res[4 * j + 2])
            history.append(res)
            j_done = j + 1
            if res <= tol or it >= max_iter or hn == 0.0:
                break
        torch.cuda.synchronize(dev)
        Hh = st[:o_g].view(m + 1, m).cpu().numpy()
        gh = st[o_g:o_g + m + 1].cpu().numpy()
        y = np.zeros(j_done, dtype=np.complex128)
        for i in range(j_done - 1, -1, -1):
            y[i] = (gh[i] - Hh[i, i + 1:j_done] @ y[i + 1:j_done]) / Hh[i, i]
        hv[:j_done] = torch.from_numpy(-y)
        _abi.check(L.h2b_zgemv_sub(ptr(V), n, j_done, ptr(hv), ptr(x), n, None, sh), "h2b_zgemv_sub")
        op.matvec_local(x, out=tmp)
        r.copy_(b)
        _abi.check(L.h2b_zaxpby(n, -1.0, 0.0, ptr(tmp), 1.0, 0.0, ptr(r), sh), "h2b_zaxpby")  # r = b - A x
        true_res = op.norm(r) / bnrm
        if true_res <= tol:
            converged = True
            break
    return x, SolveReport(it, history, converged, time.perf_counter() - t0)


def _dist_gmres_host(op, b_local, tol, restart, max_iter):
    """The same recurrence on torch CPU tensors, for the CPU plan interpreter of the tests."""
    import torch
    t0 = time.perf_counter()
    b = b_local.to(op.device, torch.complex128)
    bnrm = op.norm(b)
    if bnrm == 0.0:
        return torch.zeros_like(b), SolveReport(0, [], True, time.perf_counter() - t0)
    m = int(restart)
    x = torch.zeros_like(b)
    r = b.clone()
    V = torch.zeros((m + 1, op.nrows), dtype=torch.complex128, device=op.device)
    it, history, converged = 0, [], False
    while it < max_iter:
        beta = op.norm(r)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        for j in range(m):
            w = op.matvec_local(V[j])
            it += 1
            Vj = V[:j + 1]
            h = _multi_dot(op, Vj, w)                                      # CGS pass 1
            w = w - (h.unsqueeze(1) * Vj).sum(0)
            h2 = _multi_dot(op, Vj, w)                                     # CGS pass 2
            w = w - (h2.unsqueeze(1) * Vj).sum(0)
            hh = (h + h2).cpu().numpy()
            hn = op.norm(w)
            for i in range(j):
                a_, bb = hh[i], hh[i + 1]
                hh[i] = cs[i] * a_ + sn[i] * bb
                hh[i + 1] = -np.conj(sn[i]) * a_ + cs[i] * bb
            c, s, rr = _givens(hh[j], hn)
            cs[j], sn[j] = c, s
            H[:j + 1, j] = hh[:j + 1]
            H[j, j] = rr
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            res = abs(g[j + 1]) / bnrm
            history.append(float(res))
            j_done = j + 1
            if res <= tol:
                break
            if it >= max_iter or hn == 0.0:
                break
            V[j + 1] = w / hn
        y = np.zeros(j_done, dtype=np.complex128)
        for i in range(j_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:j_done]) / H[i, i]
        yt = torch.from_numpy(y).to(op.device)
        x = x + (yt.unsqueeze(1) * V[:j_done]).sum(0)
        r = b - op.matvec_local(x)
        true_res = op.norm(r) / bnrm
        if true_res <= tol:
            converged = True
            break
    return x, SolveReport(it, history, converged, time.perf_counter() - t0)


def _multi_dot(op, Vj, w):
    """h_i = Σ conj(V_i) w over all ranks, one all-reduce for all i."""
    import torch
    h = (Vj.conj() * w.unsqueeze(0)).sum(1)
    if op.world > 1:
        h = torch.view_as_complex(op.allreduce_(torch.view_as_real(h).clone()))
    return h
