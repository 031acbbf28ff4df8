"""Subtree-partitioned multi-GPU path: partition, shard plans, exchange and
distributed GMRES, checked on CPU — plans interpreted by oracle/plan_exec.py, collectives on
gloo with world_size 2 and 4 — against the H² oracle (pinned to the reference)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden, rel

NAMES = ["rod164", "cube8", "plate32", "line2048", "random137", "cube8_rand_eps"]


def _cvec(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _max_ranks(pk):
    from paper_1703_01175_b200.shard import partition
    out = [1]
    for G in (2, 4, 8):
        try:
            partition(pk, G)
            out.append(G)
        except ValueError:
            break
    return out


def _simulated(pk, G, X):
    """All ranks of a G-way partition run in one process; the all-gather is a copy."""
    from oracle.plan_exec import NumpyPlanEngine
    from paper_1703_01175_b200.shard import (PH_COUPLE, PH_DOWN, PH_NEAR, PH_UP_OWN, PH_UP_TOP,
                                             partition, plan_shard)
    part = partition(pk, G)
    q = X.shape[1]
    plans = [plan_shard(pk, G, g, part) for g in range(G)]
    eng = [NumpyPlanEngine(p) for p in plans]
    bufs = []
    for g, p in enumerate(plans):
        xb = torch.zeros((part.xlen, q), dtype=torch.complex128)
        xb[g * part.chunk:g * part.chunk + p.nrows] = torch.from_numpy(X[p.row0:p.row0 + p.nrows])
        bufs.append((xb, torch.zeros_like(xb), torch.zeros((p.nrows, q), dtype=torch.complex128)))
        eng[g].run(PH_UP_OWN, *bufs[g], q)
    ch = part.chunk
    gathered = torch.cat([b[0][g * ch:(g + 1) * ch] for g, b in enumerate(bufs)])
    Y = np.zeros_like(X)
    for g, p in enumerate(plans):
        bufs[g][0][:G * ch] = gathered
        for ph in (PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
            eng[g].run(ph, *bufs[g], q)
        Y[p.row0:p.row0 + p.nrows] = bufs[g][2].numpy()
    return Y


@pytest.mark.parametrize("name", NAMES)
def test_partition_covers_rows_and_skeletons(name):
    from paper_1703_01175_b200.shard import partition
    pk, _ = load_golden(name)
    for G in _max_ranks(pk):
        part = partition(pk, G)
        assert part.row0[0] == 0 and np.all(part.row0[1:] == part.row0[:-1] + part.nrows[:-1])
        assert part.row0[-1] + part.nrows[-1] == pk.n
        assert part.nrows.max() - part.nrows.min() <= 1 or G == 1 or pk.c_size.max() != pk.c_size.min()
        hats = part.hat[pk.c_rank > 0]
        assert len(np.unique(hats)) == hats.size  # every skeleton has its own exchange rows
        for c in np.nonzero(pk.c_rank > 0)[0]:
            o = part.owner[c]
            lo, hi = (o * part.chunk + part.nmax, (o + 1) * part.chunk) if o >= 0 else \
                (G * part.chunk, part.xlen)
            assert lo <= part.hat[c] and part.hat[c] + pk.c_rank[c] <= hi


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("q", [1, 3])
def test_sharded_plans_reproduce_oracle(name, q):
    from oracle import h2_oracle as ho
    pk, ex = load_golden(name)
    X = _cvec(np.random.default_rng(q), (pk.n, q))
    ref = ho.matvec_perm(pk, X)
    for G in _max_ranks(pk):
        assert rel(_simulated(pk, G, X), ref) <= 1e-13, G


def test_sharded_plan_rejects_bad_rank_counts():
    from paper_1703_01175_b200.shard import partition
    pk, _ = load_golden("rod164")
    with pytest.raises(ValueError):
        partition(pk, 3)
    with pytest.raises(ValueError):
        partition(pk, 1 << 12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["OMP_NUM_THREADS"] = "1"
    torch.set_num_threads(1)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from conftest import load_golden as lg
        from oracle.plan_exec import NumpyPlanEngine
        from paper_1703_01175_b200.dist import DistH2Operator, dist_gmres_solve
        pk, ex = lg(name)
        op = DistH2Operator(pk, engine=NumpyPlanEngine)
        xp = ex["x"][pk.perm, 0]
        X3 = np.random.default_rng(9).standard_normal((pk.n, 3)) + 0j
        sl = slice(op.row0, op.row0 + op.nrows)
        y = op.matvec_local(torch.from_numpy(xp[sl].copy())).numpy()
        Y3 = op.matvec_local(torch.from_numpy(X3[sl].copy())).numpy()
        bp = ex["bicg_rhs"][pk.perm] if "bicg_rhs" in ex else xp
        xs, rep = dist_gmres_solve(op, torch.from_numpy(bp[sl].copy()), tol=1e-8, restart=20, max_iter=400)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), y=y, Y3=Y3, xs=xs.numpy(), row0=op.row0,
                 it=rep.iterations, conv=rep.converged)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("rod164", 2), ("plate32", 2), ("cube8", 4)])
def test_gloo_distributed_matvec_and_gmres(name, world, tmp_path):
    from oracle import h2_oracle as ho
    from oracle import krylov_oracle as ko
    pk, ex = load_golden(name)
    mp.start_processes(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    parts.sort(key=lambda z: int(z["row0"]))
    y = np.concatenate([z["y"] for z in parts])
    Y3 = np.concatenate([z["Y3"] for z in parts])
    xs = np.concatenate([z["xs"] for z in parts])
    xp = ex["x"][pk.perm, 0]
    assert rel(y, ex["y"][pk.perm, 0]) <= 1e-12          # the reference's own matvec output
    X3 = np.random.default_rng(9).standard_normal((pk.n, 3)) + 0j
    assert rel(Y3, ho.matvec_perm(pk, X3)) <= 1e-12
    bp = ex["bicg_rhs"][pk.perm] if "bicg_rhs" in ex else xp
    _, ro = ko.gmres_solve(lambda v: ho.matvec_perm(pk, v), bp, tol=1e-8, restart=20, max_iter=400)
    its = {int(z["it"]) for z in parts}
    assert len(its) == 1 and abs(its.pop() - ro.iterations) <= 1
    assert all(bool(z["conv"]) for z in parts)
    assert np.linalg.norm(ho.matvec_perm(pk, xs) - bp) / np.linalg.norm(bp) <= 1e-8


@pytest.mark.parametrize("name", ["cube8", "plate32", "random137"])
def test_shard_couple_panels_reproduce_oracle(name):
    """Coupling rows as gathered panels (h2b SEG_GATHER) give the same matvec."""
    from oracle import h2_oracle as ho
    from oracle.plan_exec import NumpyPlanEngine
    from paper_1703_01175_b200.shard import PH_COUPLE, PH_DOWN, PH_NEAR, PH_UP_OWN, PH_UP_TOP, plan_shard
    pk, _ = load_golden(name)
    X = _cvec(np.random.default_rng(2), (pk.n, 2))
    plan = plan_shard(pk, 1, 0, couple_panels=True)
    assert plan.gather.size > 0
    eng = NumpyPlanEngine(plan)
    xb = torch.zeros((plan.part.xlen, 2), dtype=torch.complex128)
    xb[:pk.n] = torch.from_numpy(X)
    yh, y = torch.zeros_like(xb), torch.zeros((pk.n, 2), dtype=torch.complex128)
    for ph in (PH_UP_OWN, PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR):
        eng.run(ph, xb, yh, y, 2)
    assert rel(y.numpy(), ho.matvec_perm(pk, X)) <= 1e-13


def test_structure_exact_shards_match_oracle_on_host(tmp_path):
    """Structure-exact operator (seeded far field, near-field from geometry): shard plans built
    for the CPU interpreter reproduce the oracle on the same payloads."""
    from oracle import h2_oracle as ho
    from paper_1703_01175_b200.pack import load_packed, save_structure
    pk0, _ = load_golden("cube8")
    geom = dict(kind="lattice", dims=[8, 8, 8], h=1 / 16, eps_r=4.0, k0=2 * np.pi)
    save_structure(pk0, tmp_path / "s.npz", geom, seed=5)
    pk = load_packed(tmp_path / "s.npz")  # host payloads (the generator's values)
    bare = load_packed(tmp_path / "s.npz", near_on_host=False, far_on_host=False)
    X = _cvec(np.random.default_rng(1), (pk.n, 2))
    ref = ho.matvec_perm(pk, X)
    for G in (1, 2, 4):
        assert rel(_simulated(bare, G, X), ref) <= 1e-13, G


def test_synthetic_generator_is_counter_based():
    from paper_1703_01175_b200.synthetic import synth_values
    a = synth_values(3, 2, 0, 1000, 0.5)
    assert np.array_equal(a[100:200], synth_values(3, 2, 100, 100, 0.5))  # position-determined
    assert not np.array_equal(a, synth_values(4, 2, 0, 1000, 0.5))
    assert np.abs(a.real).max() <= 0.5 and np.abs(a.imag).max() <= 0.5
