"""Multi-GPU host logic on CPU: the subtree partition is valid, and the
fan-in algorithm the GPU ranks run (own subtrees + contributions into a local
top copy -> sum-reduce of the top region -> top on rank 0) reproduces the
sequential factor.  world_size 2 over gloo on 127.0.0.1, arithmetic by the
oracle (test infrastructure)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import panel_oracle as O
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
from paper_1405_2636_b200.distributed import (check_partition, entry_owner_mask, partition,
                                              subtree_flops, top_range)
from paper_1405_2636_b200.symbolic import PanelStore, assembly_positions


@pytest.mark.parametrize("dims,nparts", [((2, (32, 32)), 2), ((3, (10, 10, 10)), 2),
                                         ((3, (12, 12, 12)), 4), ((3, (16, 16, 16)), 8),
                                         ((3, (24, 24, 24)), 8)])
def test_partition_valid_and_balanced(dims, nparts):
    A = sparse.gen_laplacian(*dims)
    an = analyze(A)
    g = partition(an.symbol, nparts)
    check_partition(an.symbol, g)
    assert set(np.unique(g)) <= set(range(-1, nparts))
    sub = subtree_flops(an.symbol)
    own = np.zeros(nparts)
    par = an.symbol.panel_parent()
    for p in range(an.symbol.npanels):
        if g[p] >= 0 and (par[p] < 0 or g[par[p]] < 0):
            own[g[p]] += sub[p]
    assert (own > 0).sum() == min(nparts, (own > 0).sum())
    # deterministic
    assert np.array_equal(g, partition(an.symbol, nparts))


def _rank_factor(rank, world, an, group, form, thr):
    """Rank-local phase 0 on the host (oracle arithmetic)."""
    sym = an.symbol
    store = PanelStore(sym)
    pos, sel = assembly_positions(sym, an.A_perm)
    mine = entry_owner_mask(sym, an.A_perm, group, rank)
    store.slab[pos[mine]] = an.A_perm.values[sel][mine]
    for p in range(sym.npanels):
        if group[p] != rank:
            continue
        O.factor_panel(store.data[p], int(sym.starts[p]), form, thr)
        for q, blocks in O.couples_of(sym, p).items():
            O.update_couple(sym, store, p, q, blocks, form)
    return store


def _worker(rank, world, port, form, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = sparse.gen_laplacian(3, (12, 12, 12))
        if form == "ldlt":
            A = sparse.shift_diagonal(A, 0.5)
        an = analyze(A, AnalyzeOptions(form=form))
        sym = an.symbol
        group = partition(sym, world, form)
        thr = O.pivot_threshold(an.A_perm)
        store = _rank_factor(rank, world, an, group, form, thr)
        lo, hi = top_range(sym, group)
        top = torch.from_numpy(store.slab[lo:hi].copy())
        dist.reduce(top, dst=0, op=dist.ReduceOp.SUM)          # fan-in
        full = torch.from_numpy(store.slab.copy())
        full[lo:hi] = top if rank == 0 else 0
        if rank == 0:
            store.slab[lo:hi] = top.numpy()
            for p in range(sym.npanels):                        # the top on rank 0
                if group[p] >= 0:
                    continue
                O.factor_panel(store.data[p], int(sym.starts[p]), form, thr)
                for q, blocks in O.couples_of(sym, p).items():
                    O.update_couple(sym, store, p, q, blocks, form)
            full = torch.from_numpy(store.slab.copy())
        else:
            full[lo:hi] = 0
        dist.reduce(full, dst=0, op=dist.ReduceOp.SUM)         # gather owned panels
        if rank == 0:
            ref = O.factor_analysis(an)
            err = float(np.abs(full.numpy() - ref.slab).max() / np.abs(ref.slab).max())
            with open(result_path, "w") as fh:
                fh.write(repr(err))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("form", ["llt", "ldlt"])
def test_fanin_algorithm_gloo_world2(tmp_path, form):
    out = str(tmp_path / "err.txt")
    mp.spawn(_worker, args=(2, _free_port(), form, out), nprocs=2, join=True)
    err = float(open(out).read())
    assert err <= 1e-12, err


def test_top_owners_cover_and_balance():
    """Every top panel has exactly one owner; LPT keeps the owners' loads
    within the heaviest single panel of each other."""
    from paper_1405_2636_b200.distributed import partition, top_owners
    from paper_1405_2636_b200.flops import block_flops_array, factor_flops_array
    an = analyze(sparse.gen_laplacian(3, (14, 14, 14)))
    sym = an.symbol
    for world in (2, 3, 4):
        group = partition(sym, world)
        own = top_owners(sym, group, world)
        top = group < 0
        assert (own[top] >= 0).all() and (own[top] < world).all() and (own[~top] == -1).all()
        work = factor_flops_array(sym).astype(float)
        src = np.repeat(np.arange(sym.npanels), np.diff(sym.blkptr))
        sel = top[src]
        np.add.at(work, sym.blk_facing[sel], block_flops_array(sym).astype(float)[sel])
        loads = np.array([work[top & (own == r)].sum() for r in range(world)])
        assert loads.max() - loads.min() <= work[top].max() + 1e-9


def _worker_p2p(rank, world, port, form, result_path):
    """The peer-to-peer protocol of DistributedFactorizer(transport="p2p") on
    the host: phase 0, owner-side fan-in of exactly fanin_plan's segments (in
    rank order), per top level owners factor, readers pull pull_plan's
    segments, owners of destinations update; peers' slabs are read through
    all_gather (the GPU path maps them with CUDA IPC)."""
    from paper_1405_2636_b200.distributed import (fanin_plan, panel_levels, pull_plan,
                                                  top_owners)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = sparse.gen_laplacian(3, (12, 12, 12))
        if form == "ldlt":
            A = sparse.shift_diagonal(A, 0.5)
        an = analyze(A, AnalyzeOptions(form=form))
        sym = an.symbol
        group = partition(sym, world, form)
        owner = top_owners(sym, group, world, form)
        thr = O.pivot_threshold(an.A_perm)
        store = _rank_factor(rank, world, an, group, form, thr)

        def peers():
            t = torch.from_numpy(store.slab.copy())
            allt = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            return [x.numpy() for x in allt]

        slabs = peers()                                           # after phase 0
        for r, segs in fanin_plan(sym, group, owner, rank).items():
            for a, n in segs:
                store.slab[a:a + n] += slabs[r][a:a + n]
        lev = panel_levels(sym)
        top = np.flatnonzero(group < 0)
        levels = sorted({int(lev[p]) for p in top})
        pulls = pull_plan(sym, group, owner, rank, set(levels))
        for L in levels:
            mine = [p for p in top if lev[p] == L and owner[p] == rank]
            for p in mine:
                O.factor_panel(store.data[p], int(sym.starts[p]), form, thr)
            slabs = peers()
            for o, segs in pulls.get(L, {}).items():
                for a, n in segs:
                    store.slab[a:a + n] = slabs[o][a:a + n]
            for p in top:
                if lev[p] != L:
                    continue
                for q, blocks in O.couples_of(sym, p).items():
                    if owner[q] == rank:
                        O.update_couple(sym, store, p, q, blocks, form)
        full = torch.from_numpy(store.slab.copy())
        off = sym.storage_offsets()
        for p in top:
            if owner[p] != rank:
                full[off[p]:off[p + 1]] = 0
        dist.all_reduce(full, op=dist.ReduceOp.SUM)
        if rank == 0:
            ref = O.factor_analysis(an)
            err = float(np.abs(full.numpy() - ref.slab).max() / np.abs(ref.slab).max())
            with open(result_path, "w") as fh:
                fh.write(repr(err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("form,world", [("llt", 2), ("llt", 3), ("ldlt", 2)])
def test_p2p_protocol_gloo(tmp_path, form, world):
    out = str(tmp_path / "err.txt")
    mp.spawn(_worker_p2p, args=(world, _free_port(), form, out), nprocs=world, join=True)
    err = float(open(out).read())
    assert err <= (1e-12 if form == "llt" else 1e-10), err


def test_p2p_plans_move_less_than_collectives():
    """Exact fan-in pulls never exceed the dense all-reduce volume and pulls
    never exceed the broadcast volume; every needed panel is pulled once."""
    from paper_1405_2636_b200.distributed import (fanin_plan, panel_levels, pull_plan,
                                                  top_owners, top_readers)
    an = analyze(sparse.gen_laplacian(3, (16, 16, 16)))
    sym = an.symbol
    off = sym.storage_offsets()
    for world in (2, 4):
        group = partition(sym, world)
        owner = top_owners(sym, group, world)
        top = np.flatnonzero(group < 0)
        lev = panel_levels(sym)
        levels = {int(lev[p]) for p in top}
        region = sum(int(off[p + 1] - off[p]) for p in top)
        fan = pull = 0
        for r in range(world):
            fan += sum(n for segs in fanin_plan(sym, group, owner, r).values() for _, n in segs)
            pl = pull_plan(sym, group, owner, r, levels)
            pull += sum(n for d in pl.values() for segs in d.values() for _, n in segs)
        assert fan <= (world - 1) * region
        readers = top_readers(sym, group, owner)
        need = sum(int(off[p + 1] - off[p]) * len(readers.get(p, set()) - {int(owner[p])})
                   for p in top)
        assert pull == need <= (world - 1) * region
