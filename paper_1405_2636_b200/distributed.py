"""Multi-GPU numeric factorization: subtree partition + fan-in.

One process per GPU (torch.distributed, NCCL).  The panel tree is cut by
proportional mapping: the heaviest subtree is split until every candidate is
at most 1/G of the candidates' work, then candidates are LPT-packed onto the
G ranks (`partition`).  Panels above the cut form the shared *top*.

Rank r factors its own subtrees (level-batched, phase 0 of its plan) and
applies its couples into top panels to its local copy of the top
(zero-initialized, or A's values on rank 0) - the paper's fan-in
accumulation.  The top region of the slabs is then
sum-reduced onto rank 0 (one NCCL reduce: every non-top entry in that range
is owned by exactly one rank and zero elsewhere), and rank 0 factors the
top (phase 1).  The partition is pure host logic, so it is tested on CPU
(tests/test_distributed_cpu.py, gloo, world_size 2) together with the
fan-in algorithm itself (on the oracle).
"""

from __future__ import annotations

import numpy as np

from .flops import LDLT, LLT


def panel_parents(symbol):
    return symbol.panel_parent()


def subtree_flops(symbol, form=LLT):
    """Flops of each panel's subtree (factor + update tasks of the reference model)."""
    from .flops import block_flops_array, factor_flops_array
    own = factor_flops_array(symbol, form).astype(np.float64)
    owner = np.repeat(np.arange(symbol.npanels), np.diff(symbol.blkptr))
    np.add.at(own, owner, block_flops_array(symbol, form).astype(np.float64))
    par = panel_parents(symbol)
    sub = own.copy()
    for p in range(symbol.npanels):  # children precede parents
        if par[p] >= 0:
            sub[par[p]] += sub[p]
    return sub


def partition(symbol, nparts, form=LLT, keep_frac=0.3):
    """group[p] in [0, nparts) for subtree panels, -1 for the shared top.

    Deterministic (ties by panel id).  Splits stop when there are >= 2*nparts
    candidates none heavier than 1/nparts of their total, or when the
    candidates would hold less than `keep_frac` of the work.
    """
    npn = symbol.npanels
    group = np.full(npn, -1, dtype=np.int32)
    if nparts <= 1 or npn == 0:
        if nparts == 1:
            group[:] = 0
        return group
    par = panel_parents(symbol)
    kids = [[] for _ in range(npn)]
    for p in range(npn):
        if par[p] >= 0:
            kids[par[p]].append(p)
    sub = subtree_flops(symbol, form)
    cand = [p for p in range(npn) if par[p] < 0]
    total = float(sum(sub[c] for c in cand))
    while cand:
        best = max(range(len(cand)), key=lambda k: (sub[cand[k]], -cand[k]))
        csum = float(sum(sub[c] for c in cand))
        if len(cand) >= 2 * nparts and sub[cand[best]] <= csum / nparts:
            break
        if csum < keep_frac * total:
            break
        c = cand[best]
        if not kids[c]:
            break
        cand.pop(best)
        cand.extend(kids[c])
    cand.sort(key=lambda c: (-sub[c], c))
    load = np.zeros(nparts)
    root_group = {}
    for c in cand:
        g = int(np.argmin(load))
        load[g] += sub[c]
        root_group[c] = g
    for p in range(npn - 1, -1, -1):
        if p in root_group:
            group[p] = root_group[p]
        elif par[p] >= 0 and group[par[p]] >= 0:
            group[p] = group[par[p]]
    return group


def check_partition(symbol, group):
    """Couples never cross groups; group panels' ancestors are in the group or the top."""
    par = panel_parents(symbol)
    for p in range(symbol.npanels):
        if group[p] >= 0 and par[p] >= 0 and group[par[p]] not in (-1, group[p]):
            raise AssertionError(f"panel {p}: parent in another group")
        if group[p] == -1 and par[p] >= 0 and group[par[p]] >= 0:
            raise AssertionError(f"top panel {p} below a group panel")
    owner = np.repeat(np.arange(symbol.npanels), np.diff(symbol.blkptr))
    gs, gq = group[owner], group[symbol.blk_facing]
    bad = (gs >= 0) & (gq >= 0) & (gs != gq)
    if bad.any():
        raise AssertionError("a couple crosses two groups")
    return True


def top_range(symbol, group):
    """[lo, hi) slab element range holding every top panel (hi = slab end)."""
    off = symbol.storage_offsets()
    top = np.flatnonzero(group < 0)
    if not len(top):
        return int(off[-1]), int(off[-1])
    return int(off[top.min()]), int(off[-1])


def entry_owner_mask(symbol, A_perm, group, rank):
    """Lower entries of A assembled by `rank`: its own panels (+ the top on rank 0)."""
    cols = np.repeat(np.arange(A_perm.n, dtype=np.int64), np.diff(A_perm.colptr))
    lower = A_perm.rowidx >= cols
    g = group[symbol.col2panel[cols[lower]]]
    mine = (g == rank) | ((g < 0) & (rank == 0))
    return mine


def panel_levels(symbol):
    """Height of each panel in the panel tree (the level schedule's batches)."""
    par = panel_parents(symbol)
    lev = np.zeros(symbol.npanels, dtype=np.int64)
    for p in range(symbol.npanels):  # children precede parents
        if par[p] >= 0 and lev[par[p]] < lev[p] + 1:
            lev[par[p]] = lev[p] + 1
    return lev


def top_owners(symbol, group, world, form=LLT):
    """Owner rank of every top panel (-1 elsewhere): LPT over the top panels by
    their work on the owner - factor flops plus every update into them from
    top panels (the fan-in from the subtrees arrives by the all-reduce)."""
    from .flops import block_flops_array, factor_flops_array
    top = group < 0
    owner = np.full(symbol.npanels, -1, dtype=np.int32)
    if not top.any():
        return owner
    work = factor_flops_array(symbol, form).astype(np.float64)
    src = np.repeat(np.arange(symbol.npanels), np.diff(symbol.blkptr))
    bf = block_flops_array(symbol, form).astype(np.float64)
    sel = top[src]
    np.add.at(work, symbol.blk_facing[sel], bf[sel])
    load = np.zeros(world)
    for q in sorted(np.flatnonzero(top), key=lambda q: (-work[q], q)):
        r = int(np.argmin(load))
        owner[q] = r
        load[r] += work[q]
    return owner


class DistributedFactorizer:
    """One rank of a G-GPU factorization (torch.distributed must be initialized).

    distribute_top=False: the top is reduced onto rank 0 and factored there.
    distribute_top=True: every top panel has an owner rank (top_owners); after
    an all-reduce of the top region, each top level is factored by the owners,
    its panels broadcast from their owners, and the updates from that level
    applied by the owners of their destinations (the top separators split over
    all GPUs - SURVEY §8(e))."""

    def __init__(self, analysis, rank, world, device, pg=None, distribute_top=False):
        import torch
        from .engine import Engine
        self.an = analysis
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        self.pg = pg
        sym = analysis.symbol
        self.group = partition(sym, world, analysis.options.form)
        check_partition(sym, self.group)
        self.distribute_top = bool(distribute_top) and world > 1
        self.owner = top_owners(sym, self.group, world, analysis.options.form) \
            if self.distribute_top else None
        self.engine = Engine(sym, self.device, partition=(self.group, world, rank),
                             top_owner=self.owner)
        if self.distribute_top:
            self.bounds, self.seg_levels = self.engine.segments()
            lev = panel_levels(sym)
            off = sym.storage_offsets()
            top = np.flatnonzero(self.group < 0)
            self.level_panels = {}
            for p in top:
                self.level_panels.setdefault(int(lev[p]), []).append(int(p))
            self.offsets = off
        self.lo, self.hi = top_range(sym, self.group)
        self.mask = entry_owner_mask(sym, analysis.A_perm, self.group, rank)
        from .pipeline import default_pivot_threshold
        self.thr = default_pivot_threshold(analysis.A_perm)
        self.store = self.engine.new_store()
        from .symbolic import assembly_positions
        pos, sel = assembly_positions(sym, analysis.A_perm)
        self.dpos = torch.from_numpy(pos[self.mask]).to(self.device)
        vals = analysis.A_perm.values[sel][self.mask]
        self.dvals = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(self.device)

    def assemble(self, stream=None):
        self.engine.assemble_positions(self.store, self.dpos, self.dvals, stream=stream)

    def factor(self, stream=None):
        """Phase 0, fan-in reduce of the top region onto rank 0, phase 1 on rank 0."""
        import torch
        import torch.distributed as dist
        form = self.an.options.form
        self.engine.factor(self.store, form, self.thr, stream=stream, phase=0)
        if self.distribute_top:
            if self.hi > self.lo:
                dist.all_reduce(self.store[self.lo:self.hi], op=dist.ReduceOp.SUM, group=self.pg)
            b = self.bounds
            for k in range(len(b) - 1):
                self.engine.factor_range(self.store, form, self.thr, b[k], b[k + 1], stream=stream)
                if k % 2 == 0:  # level factored by the owners: broadcast its panels
                    for p in self.level_panels.get(int(self.seg_levels[k]), []):
                        o0, o1 = int(self.offsets[p]), int(self.offsets[p + 1])
                        dist.broadcast(self.store[o0:o1], src=int(self.owner[p]), group=self.pg)
            self.engine.status_all(stream=stream)
            return
        if self.hi > self.lo:
            top = self.store[self.lo:self.hi]
            if dist.get_backend(self.pg) == "nccl":
                dist.reduce(top, dst=0, op=dist.ReduceOp.SUM, group=self.pg)
            else:  # gloo (tests: several ranks sharing one GPU) has no CUDA reduce
                dist.all_reduce(top, op=dist.ReduceOp.SUM, group=self.pg)
        if self.rank == 0:
            self.engine.factor(self.store, form, self.thr, stream=stream, phase=1)

    def check(self, stream=None):
        """Raise the reference's exception if any rank saw a pivot failure
        (minimum failing column over the ranks, as the sequential reference)."""
        import torch
        import torch.distributed as dist
        if not self.distribute_top:
            self.engine.check(self.an.options.form, stream)
            return
        from .errors import NotPositiveDefiniteError, SingularPivotError
        err = None
        try:
            self.engine.check(self.an.options.form, stream)
        except (NotPositiveDefiniteError, SingularPivotError) as e:
            err = e
        big = float(2 ** 62)
        t = torch.tensor([float(err.column) if err else big, err.pivot if err else 0.0],
                         dtype=torch.float64, device=self.device)
        mine = t.clone()
        dist.all_reduce(t[:1], op=dist.ReduceOp.MIN, group=self.pg)
        if t[0].item() < big:
            col = int(t[0].item())
            piv = torch.tensor([mine[1].item() if err and err.column == col else 0.0],
                               dtype=torch.float64, device=self.device)
            dist.all_reduce(piv, op=dist.ReduceOp.SUM, group=self.pg)
            cls = SingularPivotError if self.an.options.form == LDLT else NotPositiveDefiniteError
            raise cls(col, float(piv.item()))

    def gather_factor_slab(self):
        """Full factor slab on rank 0 (sum of the ranks' owned regions)."""
        import torch.distributed as dist
        full = self.store.clone()
        if self.rank != 0:
            full[self.lo:self.hi] = 0
        if dist.get_backend(self.pg) == "nccl":
            dist.reduce(full, dst=0, op=dist.ReduceOp.SUM, group=self.pg)
        else:
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=self.pg)
        return full if self.rank == 0 else None
