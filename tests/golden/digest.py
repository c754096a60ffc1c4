"""Digest of a block symbol, computed identically from the reference's object
symbol (make_golden.py) and from the array symbol (tests)."""

import hashlib

import numpy as np


def symbol_digest(starts, rowdata, blocks, perm):
    h = hashlib.sha256()
    for arr in (starts, rowdata, blocks, perm):
        h.update(np.ascontiguousarray(np.asarray(arr, dtype=np.int64)).tobytes())
    return h.hexdigest()


def array_symbol_digest(sym, perm):
    blocks = np.stack([sym.blk_fr, sym.blk_lr, sym.blk_facing, sym.blk_loc], 1) \
        if sym.block_count() else np.zeros((0, 4), dtype=np.int64)
    return symbol_digest(sym.starts, sym.rowdata, blocks, perm)
