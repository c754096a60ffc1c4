"""Symbolic factorization, supernodes, amalgamation, panel splitting, block
structure and the panel store layout.

Host side.  Same partition rules and outputs as the reference's
`pkg/src/panelsolve/symbolic.py` (find_supernodes :88-104, amalgamate
:126-199, split_panels :202-226, build_symbol :286-315, PanelStore
:318-335), but held as flat CSR arrays (starts / rowptr / rows, and
blkptr / blk_* for blocks) so 10^6-panel symbols stay cheap; `Panel` and
`Block` objects are produced on demand for code written against the
reference's object API.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from ._native import host_lib, ptr
from .errors import StructuralError
from .ordering import NONE


# ---------------------------------------------------------------------------
# column structures (small-n API; the pipeline uses the streamed native path)

class ColumnStructure:
    """Per-column sorted row indices of L (diagonal and fill included)."""

    def __init__(self, structs):
        self.structs = structs

    def __getitem__(self, j):
        return self.structs[j]

    def __len__(self):
        return len(self.structs)

    @property
    def nnz(self):
        return int(sum(len(s) for s in self.structs))


def symbolic_factorize(pattern, tree):
    """struct(j) = pattern(j)>=j  U {j}  U  (struct(c) \\ {c}) over children c.

    Materializes every column (reference symbolic.py:36-53 contract); meant
    for small matrices and tests.  Returns (ColumnStructure, nnz_L).
    """
    n = pattern.n
    kids = tree.children()
    structs = [None] * n
    for j in range(n):
        rows = pattern.col_rows(j)
        parts = [rows[rows >= j], np.array([j], dtype=np.int64)]
        parts += [structs[c][1:] for c in kids[j]]
        structs[j] = np.unique(np.concatenate(parts))
    cs = ColumnStructure(structs)
    return cs, cs.nnz


# ---------------------------------------------------------------------------
# panel partitions

class PanelSet:
    """Ordered partition of [0, n) into panels sharing a row structure.

    starts[p]..starts[p+1] are panel p's columns; rows[rowptr[p]:rowptr[p+1]]
    its off-diagonal rows (ascending).  Constructible from a list of row
    arrays, as the reference's PanelSet(starts, rows).
    """

    def __init__(self, starts, rows, rowptr=None):
        self.starts = np.asarray(starts, dtype=np.int64)
        if rowptr is None:
            lens = np.array([len(r) for r in rows], dtype=np.int64)
            self.rowptr = np.zeros(len(lens) + 1, dtype=np.int64)
            np.cumsum(lens, out=self.rowptr[1:])
            self.rowdata = (np.concatenate([np.asarray(r, dtype=np.int64) for r in rows])
                            if len(rows) else np.zeros(0, dtype=np.int64))
        else:
            self.rowptr = np.asarray(rowptr, dtype=np.int64)
            self.rowdata = np.asarray(rows, dtype=np.int64)

    @property
    def npanels(self):
        return len(self.starts) - 1

    @property
    def rows(self):
        rp, rd = self.rowptr, self.rowdata
        return [rd[rp[p]:rp[p + 1]] for p in range(self.npanels)]

    def panel_rows(self, p):
        return self.rowdata[self.rowptr[p]:self.rowptr[p + 1]]

    def widths(self):
        return np.diff(self.starts)

    def width(self, p):
        return int(self.starts[p + 1] - self.starts[p])

    def entries(self, p):
        w = self.width(p)
        return w * (w + 1) // 2 + w * int(self.rowptr[p + 1] - self.rowptr[p])

    def total_entries(self):
        w = self.widths()
        return int(np.sum(w * (w + 1) // 2 + w * np.diff(self.rowptr)))

    def col2panel(self):
        return np.repeat(np.arange(self.npanels, dtype=np.int64), self.widths())


def fundamental_supernodes(pattern, tree):
    """Streamed native symbolic factorization + supernode detection.

    Equivalent to find_supernodes(*symbolic_factorize(pattern, tree)) of the
    reference (symbolic.py:36-53, :88-104).  Returns (PanelSet, nnz_L).
    """
    lib = host_lib()
    cp = np.ascontiguousarray(pattern.colptr, dtype=np.int64)
    ri = np.ascontiguousarray(pattern.rowidx, dtype=np.int64)
    par = np.ascontiguousarray(tree.parent, dtype=np.int64)
    h = lib.psh_symbolic(pattern.n, ptr(cp), ptr(ri), ptr(par))
    try:
        sz = np.zeros(3, dtype=np.int64)
        lib.psh_symbolic_sizes(h, ptr(sz[0:1]), ptr(sz[1:2]), ptr(sz[2:3]))
        npn, nr, nnz = (int(x) for x in sz)
        starts = np.empty(npn + 1, dtype=np.int64)
        rowptr = np.empty(npn + 1, dtype=np.int64)
        rows = np.empty(max(nr, 1), dtype=np.int64)
        lib.psh_symbolic_fetch(h, ptr(starts), ptr(rowptr), ptr(rows))
    finally:
        lib.psh_symbolic_free(h)
    return PanelSet(starts, rows[:nr], rowptr), nnz


def find_supernodes(cs, tree):
    """Maximal panels from column structures (reference symbolic.py:88-104)."""
    n = len(cs)
    counts = np.array([len(cs[j]) for j in range(n)], dtype=np.int64)
    par = np.asarray(tree.parent)
    j = np.arange(n - 1)
    merge = (par[:-1] == j + 1) & (counts[:-1] == counts[1:] + 1)
    starts = np.concatenate([[0], np.flatnonzero(~merge) + 1, [n]]).astype(np.int64)
    rows = []
    for p in range(len(starts) - 1):
        s = cs[int(starts[p])]
        rows.append(s[s >= starts[p + 1]])
    return PanelSet(starts, rows)


def panel_parents(panels):
    """Panel owning each panel's first off-diagonal row (NONE for roots)."""
    rp = panels.rowptr
    has = rp[1:] > rp[:-1]
    parent = np.full(panels.npanels, NONE, dtype=np.int64)
    first = panels.rowdata[rp[:-1][has]]
    parent[has] = np.searchsorted(panels.starts, first, side="right") - 1
    return parent


def panel_depths(panels):
    """(depth to the panel-tree root, parent) per panel (symbolic.py:116-123)."""
    parent = panel_parents(panels)
    depth = np.zeros(panels.npanels, dtype=np.int64)
    par = parent.tolist()
    d = depth.tolist()
    for p in range(panels.npanels - 1, -1, -1):
        if par[p] != NONE:
            d[p] = d[par[p]] + 1
    return np.array(d, dtype=np.int64), parent


def amalgamate(panels, nnz_original, max_fill_ratio=0.12):
    """Greedy parent-child merging under a global added-fill budget.

    Same candidate order (deepest child first, then least added fill, then
    child id) and staleness rules as the reference (symbolic.py:126-199).
    Merging only moves a parent's first column down; row lists are kept.
    """
    if max_fill_ratio < 0:
        raise ValueError("max_fill_ratio must be >= 0")
    budget = max_fill_ratio * nnz_original
    npn = panels.npanels
    st = panels.starts.tolist()
    rp = panels.rowptr
    nrow = np.diff(rp).tolist()
    first = [int(panels.rowdata[rp[p]]) if nrow[p] else -1 for p in range(npn)]
    depth, parent = panel_depths(panels)
    depth = depth.tolist()
    alive = [True] * npn
    succ = list(range(1, npn)) + [NONE]
    pred = [NONE] + list(range(npn - 1))

    def fill(c, p):
        wc = st[c + 1] - st[c]
        return wc * (st[p + 1] - st[p]) + wc * (nrow[p] - nrow[c])

    def ok(c, p):
        if c == NONE or p == NONE or not alive[c] or not alive[p]:
            return False
        if st[c + 1] != st[p]:
            return False
        return nrow[c] > 0 and st[p] <= first[c] < st[p + 1]

    heap = [(-depth[c], fill(c, int(parent[c])), c, int(parent[c]))
            for c in range(npn) if parent[c] != NONE and ok(c, int(parent[c]))]
    heapq.heapify(heap)
    added = 0
    rd = panels.rowdata
    while heap:
        _, f, c, p = heapq.heappop(heap)
        if not ok(c, p) or f != fill(c, p):
            continue
        if added + f > budget + 1e-9:
            continue
        rc = rd[rp[c]:rp[c + 1]]
        outside = rc[(rc < st[p]) | (rc >= st[p + 1])]
        if len(outside) and len(np.setdiff1d(outside, rd[rp[p]:rp[p + 1]])):
            raise StructuralError("child rows escape parent structure")
        added += f
        st[p] = st[c]
        alive[c] = False
        if pred[c] != NONE:
            succ[pred[c]] = p
        pred[p] = pred[c]
        q = pred[p]
        if q != NONE and ok(q, p):
            heapq.heappush(heap, (-depth[q], fill(q, p), q, p))
        r = succ[p]
        if r != NONE and ok(p, r):
            heapq.heappush(heap, (-depth[p], fill(p, r), p, r))
    keep = np.flatnonzero(np.array(alive, dtype=bool))
    st = np.array(st, dtype=np.int64)
    new_starts = np.append(st[keep], st[-1])
    lens = rp[keep + 1] - rp[keep]
    new_rp = np.zeros(len(keep) + 1, dtype=np.int64)
    np.cumsum(lens, out=new_rp[1:])
    idx = np.repeat(rp[keep] - new_rp[:-1], lens) + np.arange(int(new_rp[-1]))
    out = PanelSet(new_starts, rd[idx], new_rp)
    if out.total_entries() - panels.total_entries() > budget + 1e-9:
        raise StructuralError("amalgamation exceeded its fill budget")
    return out


def split_panels(panels, max_width=128, top_levels=3):
    """Cut panels at depth < top_levels wider than max_width into chained
    sub-panels of max_width columns (reference symbolic.py:202-226)."""
    if max_width < 1:
        raise ValueError("max_width must be >= 1")
    depth, _ = panel_depths(panels)
    w = panels.widths()
    cut = np.flatnonzero((depth < top_levels) & (w > max_width))
    if not len(cut):
        return PanelSet(panels.starts.copy(), panels.rowdata.copy(), panels.rowptr.copy())
    starts = [0]
    rows = []
    cutset = set(cut.tolist())
    for p in range(panels.npanels):
        fc, lc = int(panels.starts[p]), int(panels.starts[p + 1])
        pr = panels.panel_rows(p)
        if p not in cutset:
            starts.append(lc)
            rows.append(pr)
            continue
        edges = list(range(fc, lc, max_width)) + [lc]
        for k in range(len(edges) - 1):
            starts.append(edges[k + 1])
            rows.append(np.concatenate([np.arange(edges[k + 1], lc, dtype=np.int64), pr]))
    return PanelSet(np.array(starts, dtype=np.int64), rows)


# ---------------------------------------------------------------------------
# block symbolic structure

@dataclass
class Block:
    """Contiguous off-diagonal row run [fr, lr) of a panel facing `facing`."""

    fr: int
    lr: int
    facing: int
    loc: int

    @property
    def height(self):
        return self.lr - self.fr


@dataclass
class Panel:
    id: int
    fc: int
    lc: int
    rows: np.ndarray
    blocks: list = field(default_factory=list)

    @property
    def width(self):
        return self.lc - self.fc

    @property
    def nrows(self):
        return self.width + len(self.rows)

    def rowmap(self):
        return np.concatenate([np.arange(self.fc, self.lc, dtype=np.int64), self.rows])


class _PanelView:
    """Sequence of Panel objects materialized on access."""

    def __init__(self, sym):
        self._sym = sym
        self._cache = {}

    def __len__(self):
        return self._sym.npanels

    def __getitem__(self, p):
        if isinstance(p, slice):
            return [self[i] for i in range(*p.indices(len(self)))]
        if p < 0:
            p += len(self)
        if not 0 <= p < len(self):
            raise IndexError(p)
        pan = self._cache.get(p)
        if pan is None:
            s = self._sym
            b0, b1 = int(s.blkptr[p]), int(s.blkptr[p + 1])
            blocks = [Block(int(s.blk_fr[b]), int(s.blk_lr[b]), int(s.blk_facing[b]),
                            int(s.blk_loc[b])) for b in range(b0, b1)]
            pan = Panel(p, int(s.starts[p]), int(s.starts[p + 1]), s.panel_rows(p), blocks)
            self._cache[p] = pan
        return pan

    def __iter__(self):
        for p in range(len(self)):
            yield self[p]


class SymbolStructure:
    """Block symbolic structure (reference symbolic.py:271-283), array form.

    Panel p: columns [starts[p], starts[p+1]); off-diagonal rows
    rows[rowptr[p]:rowptr[p+1]]; blocks blkptr[p]..blkptr[p+1] with
    (blk_fr, blk_lr, blk_facing, blk_loc).  Storage: F-order
    nrows x width per panel, rows = [fc, lc) then the off-diagonal rows.
    """

    def __init__(self, n, starts, rowptr, rows, blkptr, blk_fr, blk_lr, blk_facing,
                 blk_loc, nnz_l):
        self.n = int(n)
        self.starts = starts
        self.rowptr = rowptr
        self.rowdata = rows
        self.blkptr = blkptr
        self.blk_fr = blk_fr
        self.blk_lr = blk_lr
        self.blk_facing = blk_facing
        self.blk_loc = blk_loc
        self.nnz_l = int(nnz_l)
        self.widths = np.diff(starts)
        self.nrows_arr = self.widths + np.diff(rowptr)
        self.col2panel = np.repeat(np.arange(len(starts) - 1, dtype=np.int64), self.widths)
        self.panels = _PanelView(self)

    @property
    def npanels(self):
        return len(self.starts) - 1

    def panel_rows(self, p):
        return self.rowdata[self.rowptr[p]:self.rowptr[p + 1]]

    def block_count(self):
        return int(self.blkptr[-1])

    def max_width(self):
        return int(self.widths.max()) if self.npanels else 0

    def max_nrows(self):
        return int(self.nrows_arr.max()) if self.npanels else 0

    def storage_offsets(self):
        """Element offset of each panel in one contiguous F-order slab (+ total).
        Computed once per symbol (a cumulative sum over every panel: 1M at
        120^3) and returned read-only."""
        off = self.__dict__.get("_storage_offsets")
        if off is None:
            off = np.zeros(self.npanels + 1, dtype=np.int64)
            np.cumsum(self.widths * self.nrows_arr, out=off[1:])
            off.flags.writeable = False
            self.__dict__["_storage_offsets"] = off
        return off

    def panel_parent(self):
        """Facing panel of each panel's first block (panel-tree parent) or NONE."""
        par = np.full(self.npanels, NONE, dtype=np.int64)
        has = self.blkptr[1:] > self.blkptr[:-1]
        par[has] = self.blk_facing[self.blkptr[:-1][has]]
        return par


def build_symbol(panels):
    """Blocks = maximal runs of consecutive rows inside one facing panel
    (reference symbolic.py:286-315), vectorized."""
    n = int(panels.starts[-1])
    npn = panels.npanels
    starts, rp, R = panels.starts, panels.rowptr, panels.rowdata
    col2panel = panels.col2panel()
    T = len(R)
    pid = np.repeat(np.arange(npn, dtype=np.int64), np.diff(rp))
    facing = col2panel[R] if T else np.zeros(0, dtype=np.int64)
    head = np.ones(T, dtype=bool)
    if T > 1:
        head[1:] = (pid[1:] != pid[:-1]) | (R[1:] != R[:-1] + 1) | (facing[1:] != facing[:-1])
    bstart = np.flatnonzero(head)
    bend = np.append(bstart[1:], T)
    bp = pid[bstart]
    blk_fr = R[bstart]
    blk_lr = R[bend - 1] + 1 if T else np.zeros(0, dtype=np.int64)
    blk_facing = facing[bstart]
    width = np.diff(starts)
    blk_loc = width[bp] + (bstart - rp[bp])
    if np.any(blk_facing <= bp):
        raise StructuralError("block faces a non-later panel")
    blkptr = np.zeros(npn + 1, dtype=np.int64)
    np.cumsum(np.bincount(bp, minlength=npn)[:npn], out=blkptr[1:])
    nnz_l = panels.total_entries()
    return SymbolStructure(n, starts.copy(), rp.copy(), R.copy(), blkptr, blk_fr,
                           blk_lr, blk_facing, blk_loc, nnz_l)


# ---------------------------------------------------------------------------
# host panel store (views into one contiguous slab)

class PanelStore:
    """Per-panel F-order (width + |rows|) x width arrays (symbolic.py:318-335).

    All panels live in one contiguous float64 slab (`slab`), at
    symbol.storage_offsets(); `data[p]` are zero-copy views.  The GPU engine
    uses the same offsets for its device slab, so host and device layouts
    are identical.
    """

    def __init__(self, symbol, slab=None, dtype=np.float64):
        self.symbol = symbol
        self.offsets = symbol.storage_offsets()
        total = int(self.offsets[-1])
        if slab is None:
            slab = np.zeros(total, dtype=dtype)
        if slab.shape != (total,):
            raise ValueError("slab size does not match the symbol")
        self.slab = slab
        self.data = _SlabViews(self)
        self.rowmaps = _RowmapView(symbol)

    def panel(self, p):
        return self.data[p]

    def local_rows(self, p, global_rows):
        rm = self.rowmaps[p]
        loc = np.searchsorted(rm, global_rows)
        if np.any(loc >= len(rm)) or np.any(rm[np.minimum(loc, len(rm) - 1)] != global_rows):
            raise StructuralError(f"rows missing from panel {p} structure")
        return loc


class _SlabViews:
    # holds the slab / offsets / symbol, not the store: no reference cycle,
    # so a store's lifetime is plain reference counting
    def __init__(self, store):
        self.slab = store.slab
        self.offsets = store.offsets
        self.symbol = store.symbol

    def __len__(self):
        return self.symbol.npanels

    def __getitem__(self, p):
        sym = self.symbol
        if p < 0:
            p += sym.npanels
        o = int(self.offsets[p])
        nr, w = int(sym.nrows_arr[p]), int(sym.widths[p])
        return self.slab[o:o + nr * w].reshape((nr, w), order="F")

    def __iter__(self):
        for p in range(len(self)):
            yield self[p]


class _RowmapView:
    def __init__(self, sym):
        self._sym = sym

    def __len__(self):
        return self._sym.npanels

    def __getitem__(self, p):
        s = self._sym
        return np.concatenate([np.arange(s.starts[p], s.starts[p + 1], dtype=np.int64),
                               s.panel_rows(p)])


def assembly_positions_any(symbol, r, c):
    """Slab position of entries (r[k], c[k]) with r >= c (lower triangle):
    offset(p) + (c - fc) * nrows(p) + local row of r in panel p = panel of
    c.  Raises StructuralError when an entry has no slot (reference
    allocate_panels / local_rows, symbolic.py:329-350)."""
    r = np.asarray(r, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    p = symbol.col2panel[c]
    fc = symbol.starts[p]
    lc = symbol.starts[p + 1]
    w = lc - fc
    nr = symbol.nrows_arr[p]
    local = np.empty(len(r), dtype=np.int64)
    inside = r < lc
    local[inside] = r[inside] - fc[inside]
    out = ~inside
    if out.any():
        n1 = symbol.n + 1
        keys = np.repeat(np.arange(symbol.npanels, dtype=np.int64),
                         np.diff(symbol.rowptr)) * n1 + symbol.rowdata
        q = p[out] * n1 + r[out]
        k = np.searchsorted(keys, q)
        kk = np.minimum(k, max(len(keys) - 1, 0))
        if len(keys) == 0 or np.any(keys[kk] != q):
            raise StructuralError("rows missing from panel structure")
        local[out] = w[out] + (k - symbol.rowptr[p[out]])
    off = symbol.storage_offsets()
    return off[p] + (c - fc) * nr + local


def assembly_positions(symbol, A):
    """Slab position of every lower entry of A (and the entry mask)."""
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.colptr))
    rows = A.rowidx
    sel = rows >= cols
    return assembly_positions_any(symbol, rows[sel], cols[sel]), sel


def assembly_positions_lu(symbol, A):
    """Positions of EVERY entry of a general A in the (L slab | U slab)
    pair: lower entries at their L-slab slot, upper entries A[i, j] (i < j)
    at the U slab's slot of (j, i), offset by the slab size."""
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.colptr))
    rows = A.rowidx
    low = rows >= cols
    pos = np.empty(len(rows), dtype=np.int64)
    pos[low] = assembly_positions_any(symbol, rows[low], cols[low])
    pos[~low] = assembly_positions_any(symbol, cols[~low], rows[~low]) + \
        int(symbol.storage_offsets()[-1])
    return pos


def allocate_panels(symbol, A):
    """Zero-initialized host PanelStore with A's lower entries scattered in."""
    store = PanelStore(symbol, dtype=np.result_type(A.values.dtype, np.float64))
    pos, sel = assembly_positions(symbol, A)
    store.slab[pos] = A.values[sel]
    return store


def gather_factor(symbol, store):
    """Dense (L, d) from the store; d is the stored block diagonal."""
    n = symbol.n
    L = np.zeros((n, n))
    d = np.zeros(n)
    for p in range(symbol.npanels):
        a = store.data[p]
        rm = store.rowmaps[p]
        fc, w = int(symbol.starts[p]), int(symbol.widths[p])
        for c in range(w):
            L[rm[c:], fc + c] = a[c:, c]
            d[fc + c] = a[c, c]
    return L, d
