"""Matrices of the golden fixtures (same constructions as make_golden.py)."""

import numpy as np

from paper_1405_2636_b200 import sparse


def rand_spd(rng, n, density):
    mask = np.tril(rng.random((n, n)) < density, -1)
    vals = rng.uniform(-1.0, 1.0, (n, n)) * mask
    Ad = vals + vals.T
    Ad += np.diag(np.abs(Ad).sum(axis=1) + rng.uniform(0.5, 1.5, n))
    r, c = np.nonzero(np.tril(Ad))
    return sparse.from_coo(n, r, c, Ad[r, c], "symmetric-lower")


def small_cases():
    rng = np.random.default_rng(20240211)
    sh = sparse.shift_diagonal
    yield "lap2d_16_llt", sparse.gen_laplacian(2, (16, 16)), "llt"
    yield "lap2d_64_llt", sparse.gen_laplacian(2, (64, 64)), "llt"
    yield "lap3d_8_llt", sparse.gen_laplacian(3, (8, 8, 8)), "llt"
    yield "lap3d_8_ldlt_shift", sh(sparse.gen_laplacian(3, (8, 8, 8)), 0.5), "ldlt"
    yield "lap2d_16_ldlt_shift", sh(sparse.gen_laplacian(2, (16, 16)), 0.5), "ldlt"
    yield "rand_spd_120", rand_spd(rng, 120, 0.15), "llt"
    yield "rand_spd_60_ldlt", rand_spd(rng, 60, 0.3), "ldlt"


def small_case(name):
    for nm, A, form in small_cases():
        if nm == name:
            return A, form
    raise KeyError(name)
