"""Fill-reducing ordering: nested dissection, elimination tree, postorder.

Host side.  The heavy loops run in C++ (`csrc/ps_host.cpp`); the rules are
the reference's (`pkg/src/panelsolve/ordering.py`): BFS level-set bisection
from a pseudo-peripheral vertex, one boundary refinement pass, minimum
degree inside leaves, ties by lowest vertex index - so the permutation is
identical to the reference's (tests/test_analysis_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import host_lib, ptr

NONE = -1


@dataclass
class Permutation:
    """perm maps old index -> new index; iperm is its inverse."""

    perm: np.ndarray
    iperm: np.ndarray

    def __post_init__(self):
        self.perm = np.asarray(self.perm, dtype=np.int64)
        self.iperm = np.asarray(self.iperm, dtype=np.int64)
        if not np.array_equal(self.perm[self.iperm], np.arange(len(self.perm))):
            raise ValueError("perm and iperm are not inverses")

    @classmethod
    def identity(cls, n):
        e = np.arange(n, dtype=np.int64)
        return cls(e, e.copy())

    @classmethod
    def from_perm(cls, perm):
        perm = np.asarray(perm, dtype=np.int64)
        ip = np.empty_like(perm)
        ip[perm] = np.arange(len(perm), dtype=np.int64)
        return cls(perm, ip)

    def compose(self, first):
        """Apply `first`, then self."""
        return Permutation.from_perm(self.perm[first.perm])


@dataclass
class EliminationTree:
    parent: np.ndarray

    def __post_init__(self):
        self.parent = np.asarray(self.parent, dtype=np.int64)

    @property
    def n(self):
        return len(self.parent)

    def children(self):
        kids = [[] for _ in range(self.n)]
        for v in np.flatnonzero(self.parent != NONE).tolist():
            kids[int(self.parent[v])].append(v)
        return kids

    def roots(self):
        return np.flatnonzero(self.parent == NONE).tolist()


def nested_dissection(G, leaf_size=64):
    """(Permutation, separator sizes of the non-leaf dissection nodes)."""
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    n = G.n
    iperm = np.empty(n, dtype=np.int64)
    cap = 2 * n + 2
    seps = np.empty(cap, dtype=np.int64)
    nsep = np.zeros(1, dtype=np.int64)
    ip = np.ascontiguousarray(G.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(G.indices, dtype=np.int64)
    rc = host_lib().psh_nested_dissection(n, ptr(ip), ptr(ix), int(leaf_size),
                                          ptr(iperm), ptr(seps), cap, ptr(nsep))
    if rc != 0:
        raise RuntimeError(f"nested dissection failed ({rc})")
    perm = np.empty(n, dtype=np.int64)
    perm[iperm] = np.arange(n, dtype=np.int64)
    return Permutation(perm, iperm), seps[:int(nsep[0])].tolist()


def elimination_tree(A):
    """Elimination tree of a symmetric-lower pattern (Liu's algorithm)."""
    parent = np.empty(A.n, dtype=np.int64)
    cp = np.ascontiguousarray(A.colptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.rowidx, dtype=np.int64)
    host_lib().psh_etree(A.n, ptr(cp), ptr(ri), ptr(parent))
    return EliminationTree(parent)


def postorder(tree):
    """po[new] = old; roots and children visited in ascending order."""
    po = np.empty(tree.n, dtype=np.int64)
    par = np.ascontiguousarray(tree.parent, dtype=np.int64)
    host_lib().psh_postorder(tree.n, ptr(par), ptr(po))
    return po


def postorder_permute(tree):
    """Relabel the tree in postorder: (permutation old->new, relabeled tree)."""
    po = postorder(tree)
    perm = np.empty(tree.n, dtype=np.int64)
    perm[po] = np.arange(tree.n, dtype=np.int64)
    newp = np.full(tree.n, NONE, dtype=np.int64)
    has = tree.parent != NONE
    newp[perm[has]] = perm[tree.parent[has]]
    return Permutation.from_perm(perm), EliminationTree(newp)
