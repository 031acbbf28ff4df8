"""Shard plans of the subtree partition executed by libh2b (h2b_plan_*) on one B200.

The ranks of a G-way partition run one after another on cuda:0 and the all-gather is a
device copy (no kernel waits on another rank's kernel), so the per-rank device programs are
checked for G = 1..8 exactly as each GPU would run them; the multi-process collectives are
covered on CPU/gloo by tests/test_dist.py."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN_NAMES, load_config, load_golden, rel

pytestmark = pytest.mark.gpu


def _ranks(pk):
    from paper_1703_01175_b200.shard import partition
    out = []
    for G in (1, 2, 4, 8):
        try:
            partition(pk, G)
            out.append(G)
        except ValueError:
            break
    return out


def _run_sharded(pk, G, X, tail=False, **plan_kw):
    from paper_1703_01175_b200.dist import CudaPlanEngine
    from paper_1703_01175_b200.shard import (PH_COUPLE, PH_DOWN, PH_NEAR, PH_UP_OWN, PH_UP_TOP,
                                             partition, plan_shard)
    part = partition(pk, G)
    q = X.shape[1]
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    plans = [plan_shard(pk, G, g, part, **plan_kw) for g in range(G)]
    eng = [CudaPlanEngine(p, 0) for p in plans]
    ch = part.chunk
    bufs = []
    for g, p in enumerate(plans):
        xb = torch.zeros((part.xlen, q), dtype=torch.complex128, device=dev)
        xb[g * ch:g * ch + p.nrows] = Xd[p.row0:p.row0 + p.nrows]
        b = (xb, torch.zeros_like(xb), torch.zeros((p.nrows, q), dtype=torch.complex128, device=dev))
        eng[g].run(PH_UP_OWN, *b, q)
        bufs.append(b)
    gathered = torch.cat([b[0][g * ch:(g + 1) * ch] for g, b in enumerate(bufs)])
    Y = torch.empty_like(Xd)
    for g, p in enumerate(plans):
        bufs[g][0][:G * ch] = gathered
        if tail:  # the dist operator's tail: near-field on a second stream beside the far field
            eng[g].run_tail(*bufs[g], q)
        else:
            for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
                eng[g].run(ph, *bufs[g], q)
        Y[p.row0:p.row0 + p.nrows] = bufs[g][2]
    torch.cuda.synchronize()
    for e in eng:
        e.close()
    return Y.cpu().numpy()


@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("q", [1, 5, 64])
def test_shard_plans_on_device_match_oracle(name, q):
    from oracle import h2_oracle as ho
    pk, _ = load_golden(name)
    X = np.random.default_rng(q).standard_normal((pk.n, q)) * (1 + 0.5j)
    ref = ho.matvec_perm(pk, X)
    for G in _ranks(pk):
        assert rel(_run_sharded(pk, G, X), ref) <= 1e-12, G


@pytest.mark.parametrize("k", [1, 2])
def test_shard_plans_on_device_baseline_configs(k):
    pk, ex = load_config(k)
    xp = ex["x"][pk.perm][:, :1]
    yp = ex["y"][pk.perm][:, :1]
    for G in (1, 2, 4, 8):
        assert rel(_run_sharded(pk, G, xp), yp) <= 1e-10, G
        assert rel(_run_sharded(pk, G, xp, tail=True), yp) <= 1e-10, G


def test_dist_operator_single_rank_gmres():
    """DistH2Operator without a process group (world 1) on cuda:0: matvec and GMRES."""
    from paper_1703_01175_b200.dist import DistH2Operator, dist_gmres_solve
    pk, ex = load_config(1)
    op = DistH2Operator(pk, device=0, rank=0, world=1)
    xp = torch.from_numpy(ex["x"][pk.perm, 0].copy()).cuda()
    assert rel(op.matvec_local(xp).cpu().numpy(), ex["y"][pk.perm, 0]) <= 1e-10
    _, rep = dist_gmres_solve(op, xp, tol=1e-6, restart=30, max_iter=2000)
    assert rep.converged and abs(rep.iterations - int(ex["gmres_iters"])) <= 1


def _run_sharded_p2p(pk, G, X):
    """Fused exchange: every rank's UP_OWN kernel stores its x̂ rows straight into all ranks'
    exchange buffers (ITEM_BCAST epilogue, P2P stores on a multi-GPU box; here the G ranks'
    buffers live on one GPU) and h2b_plan_bcast_rows pushes its x slice — no all-gather."""
    from paper_1703_01175_b200.dist import CudaPlanEngine
    from paper_1703_01175_b200.shard import (PH_COUPLE, PH_DOWN, PH_NEAR, PH_UP_OWN, PH_UP_TOP,
                                             partition, plan_shard)
    part = partition(pk, G)
    q = X.shape[1]
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    plans = [plan_shard(pk, G, g, part, bcast=True) for g in range(G)]
    eng = [CudaPlanEngine(p, 0) for p in plans]
    ch = part.chunk
    bufs = [(torch.zeros((part.xlen, q), dtype=torch.complex128, device=dev),
             torch.zeros((part.xlen, q), dtype=torch.complex128, device=dev),
             torch.zeros((p.nrows, q), dtype=torch.complex128, device=dev)) for p in plans]
    for g in range(G):
        eng[g].set_peers([bufs[o][0].data_ptr() for o in range(G) if o != g])
    for g, p in enumerate(plans):
        bufs[g][0][g * ch:g * ch + p.nrows] = Xd[p.row0:p.row0 + p.nrows]
        eng[g].bcast_rows(bufs[g][0], g * ch, p.nrows, q)
        eng[g].run(PH_UP_OWN, *bufs[g], q)
    torch.cuda.synchronize()  # stands in for the barrier collective after the exchange
    Y = torch.empty_like(Xd)
    for g, p in enumerate(plans):
        for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
            eng[g].run(ph, *bufs[g], q)
        Y[p.row0:p.row0 + p.nrows] = bufs[g][2]
    torch.cuda.synchronize()
    for e in eng:
        e.close()
    return Y.cpu().numpy()


@pytest.mark.parametrize("name", ["rod164", "cube8", "line2048", "plate32", "random137"])
@pytest.mark.parametrize("q", [1, 64])
def test_fused_p2p_exchange_matches_oracle(name, q):
    from oracle import h2_oracle as ho
    pk, _ = load_golden(name)
    X = np.random.default_rng(q).standard_normal((pk.n, q)) * (1 - 0.5j)
    ref = ho.matvec_perm(pk, X)
    for G in _ranks(pk)[1:]:
        assert rel(_run_sharded_p2p(pk, G, X), ref) <= 1e-12, G


def test_ipc_exchange_buffer_view_roundtrip():
    """The raw exchange allocation (h2b_device_alloc, shareable with CUDA IPC) seen as a torch
    tensor, written by a plan broadcast into a 'peer' buffer on the same device."""
    import ctypes
    from paper_1703_01175_b200 import _abi
    from paper_1703_01175_b200.dist import _device_view
    L = _abi.lib()
    raw = ctypes.c_void_p()
    _abi.check(L.h2b_device_alloc(0, 16 * 2 * 100 * 3, ctypes.byref(raw)))
    dev = torch.device("cuda:0")
    a, b = (_device_view(raw.value + 16 * 300 * k, (100, 3), dev) for k in range(2))
    assert a.dtype == torch.complex128 and a.shape == (100, 3) and not a.any()
    a.copy_(torch.arange(300, dtype=torch.float64, device=dev).reshape(100, 3) * (1 + 1j))
    assert torch.equal(a, torch.arange(300, dtype=torch.float64, device=dev).reshape(100, 3) * (1 + 1j))
    assert not b.any()
    hd = (ctypes.c_char * 64)()
    _abi.check(L.h2b_ipc_get_handle(raw, hd))  # shareable (opened by the other ranks' processes)
    _abi.check(L.h2b_device_free(raw))


@pytest.mark.parametrize("name", ["cube8", "plate32", "random137", "line2048"])
@pytest.mark.parametrize("q", [1, 64])
def test_shard_couple_panels_on_device(name, q):
    """Coupling rows as gathered panels: GEMV (q = 1) and DMMA (q >= 2) gather paths."""
    from oracle import h2_oracle as ho
    pk, _ = load_golden(name)
    X = np.random.default_rng(7).standard_normal((pk.n, q)) * (0.5 + 1j)
    ref = ho.matvec_perm(pk, X)
    for G in _ranks(pk):
        assert rel(_run_sharded(pk, G, X, couple_panels=True), ref) <= 1e-12, G


def test_device_synthetic_generator_matches_host():
    import ctypes
    from paper_1703_01175_b200 import _abi
    from paper_1703_01175_b200.synthetic import synth_values
    buf = torch.empty(5000, dtype=torch.complex128, device="cuda")
    _abi.check(_abi.lib().h2b_fill_synthetic_raw(ctypes.c_void_p(buf.data_ptr()), 5000, 123456, 2, 77, 0.01))
    assert np.array_equal(buf.cpu().numpy(), synth_values(77, 2, 123456, 5000, 0.01))


@pytest.mark.parametrize("name,geom", [
    ("cube8", dict(kind="lattice", dims=[8, 8, 8], h=1 / 16, eps_r=4.0, k0=2 * np.pi)),
    ("plate32", dict(kind="lattice", dims=[32, 32, 1], h=1 / 16, eps_r=4.0, k0=2 * np.pi))])
def test_device_generated_shards_equal_single_gpu_operator(name, geom, tmp_path):
    """Shard payloads generated on the device (seeded far field, near-field from geometry) give
    the same operator as the single-GPU structure-exact handle, for G = 1..8 ranks."""
    from paper_1703_01175_b200 import H2Operator
    from paper_1703_01175_b200.pack import load_packed, save_structure
    pk0, _ = load_golden(name)
    save_structure(pk0, tmp_path / "s.npz", geom, seed=9)
    bare = load_packed(tmp_path / "s.npz", near_on_host=False, far_on_host=False)
    op = H2Operator(bare)
    X = np.random.default_rng(4).standard_normal((bare.n, 3)) * (1 + 0.25j)
    ref = op.matmat(X[np.argsort(bare.perm)])[bare.perm]  # permuted order
    for G in _ranks(bare):
        assert rel(_run_sharded(bare, G, X, device_payloads=True), ref) <= 1e-12, G


def _dist_gmres_worker(rank, world, port, path, out):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1703_01175_b200.dist import DistH2Operator, dist_gmres_solve
    from paper_1703_01175_b200.pack import load_packed
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pk, ex = load_packed(path, with_extra=True, near_on_host=False)
    op = DistH2Operator(pk, device=0)  # gloo: the exchange is host-staged, no rank waits in a kernel
    b = ex["rhs_plane_wave"][pk.perm]
    sl = slice(op.row0, op.row0 + op.nrows)
    xl, rep = dist_gmres_solve(op, torch.from_numpy(b[sl].copy()).cuda(), tol=1e-6, restart=50,
                               max_iter=3000)
    parts = [None] * world
    dist.all_gather_object(parts, (op.row0, xl.cpu().numpy()))
    if rank == 0:
        xp = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
        x = np.empty_like(xp)
        x[pk.perm] = xp
        np.savez(out, x=x, it=rep.iterations, conv=rep.converged, hist=np.asarray(rep.residual_history))
    dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 4])
def test_dist_gmres_ranks_on_one_gpu_match_oracle(G, tmp_path):
    """Row-distributed GMRES(50) on the reference-built plate pin, G gloo ranks sharing cuda:0
    (libh2b multi-dot / update / device Givens per rank, one all-reduce per CGS pass): iterations
    +-1 vs the oracle (= scipy) and the same solution."""
    import os
    import socket
    import torch.multiprocessing as mp
    from conftest import ROOT
    path = os.path.join(ROOT, "fixtures", "pin_plate256x128.npz")
    if not os.path.exists(path):
        pytest.skip("plate pin not present")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res.npz")
    mp.start_processes(_dist_gmres_worker, args=(G, port, path, out), nprocs=G, join=True,
                       start_method="spawn")
    from paper_1703_01175_b200.pack import load_packed
    pk, ex = load_packed(path, with_extra=True, near_on_host=False)
    r = np.load(out)
    assert bool(r["conv"])
    assert abs(int(r["it"]) - int(ex["gmres_iters"])) <= 1
    assert rel(r["x"], ex["gmres_x"]) <= 1e-5
    k = min(20, len(r["hist"]))
    assert np.allclose(r["hist"][:k], ex["gmres_hist"][:k], rtol=1e-6)
