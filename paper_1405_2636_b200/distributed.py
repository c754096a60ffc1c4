"""Multi-GPU numeric factorization: subtree partition + fan-in.

One process per GPU (torch.distributed for the plumbing).  The panel tree is
cut by proportional mapping: the heaviest subtree is split until every
candidate is at most 1/G of the candidates' work, then candidates are
LPT-packed onto the G ranks (`partition`).  Panels above the cut form the
shared *top*; every top panel has an owner rank (`top_owners`).

Rank r factors its own subtrees (level-batched, phase 0 of its plan) and
applies its couples into top panels to its local copy of the top
(zero-initialized, or A's values on rank 0) - the paper's fan-in
accumulation.  Then, with the default peer-to-peer
transport (distribute_top=True, transport="p2p"):

  * fan-in: the owner of each top panel adds, in rank order, the copies of
    exactly the peers that contributed to it, reading their slabs directly
    over NVLink (CUDA IPC mappings, ps_p2p_segment_add) - no all-reduce of
    the whole top region;
  * per top level: the owners factor their panels of that level; every rank
    that owns a destination of such a panel pulls it from the owner's slab
    (a peer copy) - no broadcast to ranks that do not need it; the owners of
    the destinations then apply the level's updates;
  * ordering is device-side: 64-bit epoch flags per rank (release stores /
    acquire spins at system scope, ps_p2p_signal / ps_p2p_wait) between the
    producer's stream and the consumer's - no host barrier on the path.

transport="nccl" keeps the previous collective design (all-reduce of the top
region, per-panel NCCL broadcasts); distribute_top=False reduces the top
onto rank 0 and factors it there.  The partition, ownership and transfer
plans are pure host logic, tested on CPU (tests/test_distributed_cpu.py,
gloo, world_size 2); the device path runs with several ranks sharing one
GPU in tests/test_gpu_distributed.py.
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


def top_contributors(symbol, group):
    """{top panel q: set of ranks whose local copy of q holds contributions}
    after phase 0: the groups of the subtree panels with a couple into q,
    plus rank 0 (A's entries of the top are assembled there)."""
    top = group < 0
    src = np.repeat(np.arange(symbol.npanels), np.diff(symbol.blkptr))
    dst = symbol.blk_facing
    sel = top[dst] & ~top[src]
    out = {int(q): {0} for q in np.flatnonzero(top)}
    for g, q in set(zip(group[src[sel]].tolist(), dst[sel].tolist())):
        out[q].add(int(g))
    return out


def top_readers(symbol, group, owner):
    """{top panel p: set of ranks owning a top destination of p} (the ranks
    that need p's factored values for the updates they apply)."""
    top = group < 0
    src = np.repeat(np.arange(symbol.npanels), np.diff(symbol.blkptr))
    dst = symbol.blk_facing
    sel = top[src] & top[dst]
    out = {}
    for p, q in set(zip(src[sel].tolist(), dst[sel].tolist())):
        out.setdefault(p, set()).add(int(owner[q]))
    return out


def _merge(segs):
    """Sorted, merged (offset, length) list."""
    out = []
    for a, n in sorted(segs):
        if out and out[-1][0] + out[-1][1] == a:
            out[-1][1] += n
        else:
            out.append([a, n])
    return [(int(a), int(n)) for a, n in out]


def fanin_plan(symbol, group, owner, rank):
    """{peer r: [(slab offset, length)]}: the top panels `rank` owns that peer
    r contributed to - what the owner adds from r's slab after phase 0."""
    off = symbol.storage_offsets()
    plan = {}
    for q, cs in top_contributors(symbol, group).items():
        if int(owner[q]) != rank:
            continue
        for r in cs - {rank}:
            plan.setdefault(r, []).append((int(off[q]), int(off[q + 1] - off[q])))
    return {r: _merge(v) for r, v in sorted(plan.items())}


def pull_plan(symbol, group, owner, rank, levels):
    """{top level L: {owner o: [(offset, length)]}}: panels of level L factored
    by another rank that `rank` needs (it owns one of their destinations)."""
    off = symbol.storage_offsets()
    lev = panel_levels(symbol)
    plan = {}
    for p, rd in top_readers(symbol, group, owner).items():
        o = int(owner[p])
        if o == rank or rank not in rd:
            continue
        L = int(lev[p])
        if L not in levels:
            continue
        plan.setdefault(L, {}).setdefault(o, []).append((int(off[p]), int(off[p + 1] - off[p])))
    return {L: {o: _merge(v) for o, v in sorted(d.items())} for L, d in plan.items()}


class PeerSlabs:
    """Every rank's slab and flag words mapped into this process through
    CUDA IPC (torch's tensor-sharing handles, exchanged once over the
    process group).  On an NVSwitch box the mappings are NVLink peer memory;
    ranks sharing one GPU (tests) map the same device's memory."""

    def __init__(self, store, flags, rank, world, pg=None):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        mine = (reduce_tensor(store), reduce_tensor(flags))
        every = [None] * world
        dist.all_gather_object(every, mine, group=pg)
        self.slabs, self.flags = [], []
        for r, ((f1, a1), (f2, a2)) in enumerate(every):
            if r == rank:
                self.slabs.append(store)
                self.flags.append(flags)
            else:
                self.slabs.append(f1(*a1))
                self.flags.append(f2(*a2))


class DistributedFactorizer:
    """One rank of a G-GPU factorization (torch.distributed must be initialized).

    distribute_top=True (every top panel has an owner rank, top_owners):
      transport="p2p" (default) - fan-in by owner-side peer reads of exactly
      the contributing slabs, per-level pulls of the factored panels by the
      ranks that need them, device-side epoch flags (module docstring);
      transport="nccl" - all-reduce of the top region, each factored panel
      broadcast to every rank.
    distribute_top=False: the top is reduced onto rank 0 and factored there."""

    FLAG_SCALE = 1 << 24      # level flag value = epoch * FLAG_SCALE + step
    WAIT_TIMEOUT_S = 120.0    # device-side waits give up (and raise) after this

    def __init__(self, analysis, rank, world, device, pg=None, distribute_top=False,
                 transport="p2p"):
        import torch
        from .engine import Engine
        if transport not in ("p2p", "nccl"):
            raise ValueError(f"unknown transport '{transport}'")
        self.an = analysis
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        self.pg = pg
        sym = analysis.symbol
        self.group = partition(sym, world, analysis.options.form)
        check_partition(sym, self.group)
        self.distribute_top = bool(distribute_top) and world > 1
        self.transport = transport if self.distribute_top else "nccl"
        self.owner = top_owners(sym, self.group, world, analysis.options.form) \
            if self.distribute_top else None
        self.engine = Engine(sym, self.device, partition=(self.group, world, rank),
                             top_owner=self.owner)
        self.offsets = sym.storage_offsets()
        if self.distribute_top:
            self.bounds, self.seg_levels = self.engine.segments()
            lev = panel_levels(sym)
            top = np.flatnonzero(self.group < 0)
            self.level_panels = {}
            for p in top:
                self.level_panels.setdefault(int(lev[p]), []).append(int(p))
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
        self.epoch = 0
        if self.transport == "p2p":
            self._setup_p2p()

    # ---- peer-to-peer transport ----
    def _setup_p2p(self):
        import torch
        sym = self.an.symbol
        # flag words: [0] phase 0 done (epoch), [1] top step done (epoch * S + k),
        # [2] done reading peers (epoch)
        self.flags = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.timeout = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.peers = PeerSlabs(self.store, self.flags, self.rank, self.world, self.pg)
        self.fanin = {}
        for r, segs in fanin_plan(sym, self.group, self.owner, self.rank).items():
            self.fanin[r] = self._segments(segs)
        levels = {int(self.seg_levels[k]) for k in range(0, len(self.bounds) - 1, 2)}
        self.pulls = pull_plan(sym, self.group, self.owner, self.rank, levels)

    def _segments(self, segs):
        import torch
        seg = np.asarray(segs, dtype=np.int64).reshape(-1, 2)
        start = np.concatenate([[0], np.cumsum(seg[:, 1])]).astype(np.int64)
        return (torch.from_numpy(seg.ravel().copy()).to(self.device),
                torch.from_numpy(start).to(self.device), len(seg), int(start[-1]))

    def _flag_ptr(self, r, k):
        import ctypes
        return ctypes.c_void_p(self.peers.flags[r].data_ptr() + 8 * k)

    def _signal(self, k, value, stream):
        from .engine import _stream_handle
        self.engine._check(self.engine.lib.ps_p2p_signal(self._flag_ptr(self.rank, k), int(value),
                                                         _stream_handle(stream)))

    def _wait(self, r, k, value, stream):
        import ctypes
        from .engine import _stream_handle
        self.engine._check(self.engine.lib.ps_p2p_wait(
            self._flag_ptr(r, k), int(value), ctypes.c_void_p(self.timeout.data_ptr()),
            float(self.WAIT_TIMEOUT_S), _stream_handle(stream)))

    def _fanin_p2p(self, e, stream):
        import ctypes
        from .engine import _stream_handle
        for r, (seg, start, nseg, total) in self.fanin.items():  # rank order: deterministic
            self._wait(r, 0, e, stream)
            self.engine._check(self.engine.lib.ps_p2p_segment_add(
                ctypes.c_void_p(self.store.data_ptr()), ctypes.c_void_p(self.peers.slabs[r].data_ptr()),
                ctypes.c_void_p(seg.data_ptr()), ctypes.c_void_p(start.data_ptr()), int(nseg),
                int(total), _stream_handle(stream)))

    def _pull_level(self, L, e, k, stream):
        import torch
        for o, segs in self.pulls.get(L, {}).items():
            self._wait(o, 1, e * self.FLAG_SCALE + k + 1, stream)
            src = self.peers.slabs[o]
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                for a, n in segs:
                    self.store[a:a + n].copy_(src[a:a + n], non_blocking=True)

    # ---- public ----
    def assemble(self, stream=None):
        if self.transport == "p2p" and self.epoch > 0:
            # peers may still read my previous factor (fan-in / pulls): wait
            # until every one of them has finished that epoch
            for r in range(self.world):
                if r != self.rank:
                    self._wait(r, 2, self.epoch, stream)
        self.engine.assemble_positions(self.store, self.dpos, self.dvals, stream=stream)

    def factor(self, stream=None):
        """Phase 0, fan-in, then the top (distributed or on rank 0)."""
        import torch
        import torch.distributed as dist
        form = self.an.options.form
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.engine.factor(self.store, form, self.thr, stream=stream, phase=0)
        if self.transport == "p2p":
            e = self.epoch = self.epoch + 1
            self._signal(0, e, stream)
            self._fanin_p2p(e, stream)
            b = self.bounds
            for k in range(len(b) - 1):
                self.engine.factor_range(self.store, form, self.thr, b[k], b[k + 1], stream=stream)
                if k % 2 == 0:  # level factored by its owners: publish, pull what I need
                    self._signal(1, e * self.FLAG_SCALE + k + 1, stream)
                    self._pull_level(int(self.seg_levels[k]), e, k, stream)
            self._signal(2, e, stream)
            self.engine.status_all(stream=stream)
            return
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
        if self.transport == "p2p":
            torch.cuda.synchronize(self.device)
            if int(self.timeout.item()):
                raise RuntimeError("multi-GPU flag wait timed out (peer rank stalled)")
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

    def close(self):
        """Release the peer mappings on every rank before any rank exits (a
        producer must outlive the consumers of its IPC handles)."""
        import gc
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        if getattr(self, "peers", None) is not None:
            self.peers = None
            gc.collect()
        dist.barrier(group=self.pg)

    def owned_ranges(self):
        """Slab (start, length) ranges of the panels final on this rank: its
        subtree panels, and the top panels it owns (distributed top) or the
        whole top on rank 0 (collective transport, top on rank 0)."""
        g = self.group
        if self.distribute_top:
            mine = (g == self.rank) | ((g < 0) & (self.owner == self.rank))
        else:
            mine = (g == self.rank) | ((g < 0) & (self.rank == 0))
        out = []
        for p in np.flatnonzero(mine):
            o0, o1 = int(self.offsets[p]), int(self.offsets[p + 1])
            if out and out[-1][0] + out[-1][1] == o0:
                out[-1][1] += o1 - o0
            elif o1 > o0:
                out.append([o0, o1 - o0])
        return [(a, b) for a, b in out]

    def host_values(self):
        """This rank's entries of A (the ones it assembles), as in dvals."""
        from .symbolic import assembly_positions
        _, sel = assembly_positions(self.an.symbol, self.an.A_perm)
        return np.ascontiguousarray(self.an.A_perm.values[sel][self.mask], dtype=np.float64)

    def gather_factor_slab(self):
        """Full factor slab on rank 0 (a sum over the ranks of what each one
        holds final)."""
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        full = self.store.clone()
        if self.transport == "p2p":
            # subtree panels live on their rank only; top panels are final on their owner
            for p in np.flatnonzero(self.group < 0):
                if int(self.owner[p]) != self.rank:
                    full[int(self.offsets[p]):int(self.offsets[p + 1])] = 0
        elif self.rank != 0:
            # collectives: after the all-reduce / broadcasts rank 0 holds the whole
            # [lo, hi) range final (subtree panels inside it included)
            full[self.lo:self.hi] = 0
        if dist.get_backend(self.pg) == "nccl":
            dist.reduce(full, dst=0, op=dist.ReduceOp.SUM, group=self.pg)
        else:
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=self.pg)
        return full if self.rank == 0 else None


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
