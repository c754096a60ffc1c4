"""analyze(): ordering, symbolic factorization, panels and block structure.

Host side of the drop-in (reference `pipeline.analyze`, pipeline.py:39-70):
the same steps and options, producing the same permuted matrix, permutation
and SymbolStructure.  The reference's task DAG (`Analysis.graph`) is not
built eagerly - the GPU engine schedules by panel-tree level instead - but
is available lazily through `taskgraph.build_taskgraph`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import flops as _flops
from . import sparse, symbolic
from .ordering import (EliminationTree, Permutation, elimination_tree,
                       nested_dissection, postorder_permute)

LLT = _flops.LLT
LDLT = _flops.LDLT
LU = _flops.LU
FORMS = (LLT, LDLT, LU)


@dataclass
class AnalyzeOptions:
    ordering: str = "nd"            # nd | natural
    nd_leaf: int = 64
    amalgamation: float = 0.12
    split_width: int = 128
    split_levels: int = 3
    form: str = LLT


@dataclass
class Analysis:
    A_perm: sparse.SparseMatrix
    perm: Permutation
    tree: EliminationTree
    symbol: symbolic.SymbolStructure
    options: AnalyzeOptions
    nnz_a: int
    nnz_l_presplit: int
    flops: int
    separator_sizes: list = field(default_factory=list)
    _graph: object = None

    @property
    def is_complex(self):
        return np.iscomplexobj(self.A_perm.values)

    @property
    def graph(self):
        if self._graph is None:
            from .taskgraph import build_taskgraph, compute_costs_and_priorities
            g = build_taskgraph(self.symbol)
            compute_costs_and_priorities(g, self.symbol, self.options.form)
            self._graph = g
        return self._graph


def analyze(A, options=None):
    """Ordering, symbolic factorization, panel construction.

    form "lu" (no reference counterpart): the ordering and
    symbol come from the pattern of A + A^T exactly as for the symmetric
    forms; A_perm keeps all of A's values (general storage, P A P^T).
    Complex values (complex128) are accepted for every form."""
    opts = options or AnalyzeOptions()
    if opts.form not in FORMS:
        raise ValueError(f"unknown form '{opts.form}'")
    S = sparse.symmetrize_pattern(A)
    if opts.ordering == "nd":
        G = sparse.adjacency_from_pattern(S)
        P0, seps = nested_dissection(G, opts.nd_leaf)
    elif opts.ordering == "natural":
        P0, seps = Permutation.identity(S.n), []
    else:
        raise ValueError(f"unknown ordering '{opts.ordering}'")
    A1 = sparse.permute_symmetric(S, P0.perm)
    tree = elimination_tree(A1)
    P1, tree = postorder_permute(tree)
    P = P1.compose(P0)
    A2 = sparse.permute_symmetric(S, P.perm)
    panels, nnz_l = symbolic.fundamental_supernodes(A2, tree)
    if opts.amalgamation > 0:
        panels = symbolic.amalgamate(panels, nnz_l, opts.amalgamation)
    presplit = panels.total_entries()
    if opts.split_width and opts.split_width > 0:
        panels = symbolic.split_panels(panels, opts.split_width, opts.split_levels)
    sym = symbolic.build_symbol(panels)
    if opts.form == LU:
        A2 = sparse.permute_general(A, P.perm)
    fl = _flops.total_flops(sym, opts.form, np.iscomplexobj(A2.values))
    return Analysis(A2, P, tree, sym, opts, S.nnz, presplit, fl, seps)
