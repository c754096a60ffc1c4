"""Parity of the CUDA engine (through the C ABI) with the oracle and with the
reference's own factors.  Tolerances: LLt factor entries <= 1e-12 relative
(max|dL|/max|L|, as reference tests/test_acceptance.py:72-73); shifted
LDLt <= 10x the reference's own sequential-vs-dynamic spread; backward
error ||Ax-b||/||b|| <= 1e-12 (north star)."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _cases import small_case, small_cases  # noqa: E402
from oracle import panel_oracle as O  # noqa: E402
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.engine import Engine  # noqa: E402
from paper_1405_2636_b200.errors import (NotPositiveDefiniteError,  # noqa: E402
                                         SingularPivotError)
from paper_1405_2636_b200.pipeline import check_solve, factorize  # noqa: E402
from paper_1405_2636_b200.symbolic import (PanelSet, PanelStore, build_symbol,  # noqa: E402
                                           gather_factor)

HERE = os.path.dirname(__file__)
SLABS = np.load(os.path.join(HERE, "golden", "factors_small.npz"))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def two_panel_symbol(width, src_rows, ndst):
    """Reference tests/test_kernels.py:86-110 one_block_setup, array form."""
    ps = PanelSet(np.array([0, width, width + ndst]),
                  [np.array(src_rows, dtype=np.int64), np.zeros(0, dtype=np.int64)])
    return build_symbol(ps)


def to_dev(store):
    return torch.from_numpy(store.slab.copy()).cuda()


# --------------------------------------------------------------------------
# task-level operators (reference plugin protocol)

def test_update_task_random_couples():
    rng = np.random.default_rng(909)
    for trial in range(60):
        width = int(rng.integers(1, 140))
        ndst = int(rng.integers(1, 150))
        k = int(rng.integers(1, ndst + 1))
        src_rows = np.sort(rng.choice(np.arange(width, width + ndst), size=k, replace=False))
        sym = two_panel_symbol(width, src_rows, ndst)
        host = PanelStore(sym)
        host.slab[:] = rng.standard_normal(host.slab.shape)
        for form in ("llt", "ldlt"):
            eng = Engine(sym)
            dev = to_dev(host)
            eng.run_update_task(dev, 0, 1, form)
            ref = PanelStore(sym, slab=host.slab.copy())
            O.update_couple(sym, ref, 0, 1, list(range(sym.blkptr[0], sym.blkptr[1])), form)
            got = dev.cpu().numpy()
            assert rel(got, ref.slab) <= 1e-13, (trial, width, ndst, form)


def test_update_task_gapped_example():
    # reference tests/test_kernels.py:146-161: rows {1,3} facing rows {1,2,3}
    sym = two_panel_symbol(1, [1, 3], 3)
    rng = np.random.default_rng(20240211)
    host = PanelStore(sym)
    host.slab[:] = rng.standard_normal(host.slab.shape)
    src = host.data[0].copy()
    dst = host.data[1].copy()
    eng = Engine(sym)
    dev = to_dev(host)
    eng.run_update_task(dev, 0, 1, "llt")
    out = PanelStore(sym, slab=dev.cpu().numpy()).data[1]
    col = src[:, 0]
    W = np.outer(col[1:], col[1:])
    expect = dst.copy()
    gl = [1, 3]
    for bi, gc in enumerate(gl):
        for ri, gr in enumerate(gl):
            if gr >= gc:
                expect[gr - 1, gc - 1] -= W[ri, bi]
    assert np.abs(out - expect).max() <= 1e-15


@pytest.mark.parametrize("w,extra", [(1, 5), (2, 3), (7, 40), (64, 130), (65, 10), (150, 300),
                                     (200, 0), (257, 129)])
@pytest.mark.parametrize("form", ["llt", "ldlt"])
def test_factor_task_vs_oracle(w, extra, form):
    rng = np.random.default_rng(w * 1000 + extra)
    n = w + extra
    M = rng.standard_normal((n, n)) / np.sqrt(n)
    Ad = M @ M.T + np.eye(n) * (2.0 if form == "llt" else 0.0)
    if form == "ldlt":
        Ad = Ad - 0.3 * np.eye(n) + np.diag(rng.choice([-3.0, 3.0], n))
    rows = np.arange(w, n, dtype=np.int64)
    ps_ = PanelSet(np.array([0, w, n]) if extra else np.array([0, w]),
                   [rows, np.zeros(0, dtype=np.int64)] if extra else [np.zeros(0, dtype=np.int64)])
    sym = build_symbol(ps_)
    host = PanelStore(sym)
    a = host.data[0]
    a[:, :] = Ad[:, :w]
    a[np.triu_indices(w, 1)] = 0.0
    eng = Engine(sym)
    dev = to_dev(host)
    eng.run_factor_task(dev, 0, form, 0.0)
    got = PanelStore(sym, slab=dev.cpu().numpy()).data[0]
    ref = a.copy(order="F")
    O.factor_panel(ref, 0, form, 0.0)
    assert rel(got, ref) <= 1e-11, (w, extra, form)
    assert np.all(got[np.triu_indices(w, 1)] == 0.0)


def test_factor_task_failure_column():
    sym = build_symbol(PanelSet(np.array([0, 3]), [np.zeros(0, dtype=np.int64)]))
    host = PanelStore(sym)
    host.data[0][:, :] = np.array([[4.0, 0, 0], [2.0, 1.0, 0], [0.0, 0.0, 1.0]])
    eng = Engine(sym)
    with pytest.raises(NotPositiveDefiniteError) as e:
        eng.run_factor_task(to_dev(host), 0, "llt", 0.0)
    assert e.value.column == 1


# --------------------------------------------------------------------------
# whole factorizations

@pytest.mark.parametrize("name,A,form", list(small_cases()), ids=lambda x: x if isinstance(x, str) else "")
def test_factorize_matches_reference_golden(name, A, form):
    an = analyze(A, AnalyzeOptions(form=form))
    res = factorize(an)
    ref = SLABS[name]
    # LLt: order-insensitive (<= 6e-16 measured); shifted indefinite LDLt
    # amplifies summation-order differences (7.3e-14 measured at 8^3)
    tol = 1e-13 if form == "llt" else 1e-12
    assert rel(res.store.slab, ref) <= tol
    r, _ = check_solve(A, res)
    assert r <= 1e-12


def test_factorize_24_cube_vs_reference():
    g = GOLD["large"]["lap3d_24_llt"]
    A = sparse.gen_laplacian(3, (24, 24, 24))
    an = analyze(A)
    res = factorize(an)
    s = res.store.slab[::g["sample_step"]]
    assert np.abs(s - np.array(g["sample"])).max() / g["max_abs_L"] <= 1e-12
    b = sparse.spmv(A, np.ones(A.n))
    x = res.solve(b)
    assert sparse.backward_error(A, x, b) <= 1e-12


def test_factorize_24_cube_ldlt_shift_vs_reference():
    g = GOLD["large"]["lap3d_24_ldlt_shift"]
    A = sparse.shift_diagonal(sparse.gen_laplacian(3, (24, 24, 24)), 0.5)
    an = analyze(A, AnalyzeOptions(form="ldlt"))
    res = factorize(an)
    s = res.store.slab[::g["sample_step"]]
    err = np.abs(s - np.array(g["sample"])).max() / g["max_abs_L"]
    assert err <= max(10 * g["self_spread"], 1e-12), err
    b = sparse.spmv(A, np.ones(A.n))
    x = res.solve(b)
    assert sparse.backward_error(A, x, b) <= 10 * max(g["backward_error"], 1e-13)


def test_random_spd_vs_dense_cholesky():
    # reference acceptance criterion 1 (tests/test_acceptance.py:60-74), seed 101
    from conftest import rand_spd
    rng = np.random.default_rng(101)
    for trial in range(20):
        n = int(rng.integers(10, 201))
        A, _ = rand_spd(rng, n, float(rng.uniform(0.05, 0.30)))
        an = analyze(A)
        res = factorize(an)
        L, _ = gather_factor(an.symbol, res.store)
        oracle = np.linalg.cholesky(an.A_perm.to_dense())
        assert np.abs(L - oracle).max() <= 1e-12 * np.abs(oracle).max(), trial


def test_wide_dense_panel():
    # one 300-wide panel: blocked factor steps + intra-panel trailing updates
    rng = np.random.default_rng(3)
    n = 300
    M = rng.standard_normal((n, n))
    Ad = M @ M.T / n + np.eye(n)
    from conftest import dense_to_lower_sparse
    A = dense_to_lower_sparse(Ad)
    an = analyze(A, AnalyzeOptions(ordering="natural", amalgamation=0, split_width=0))
    assert an.symbol.npanels == 1
    res = factorize(an)
    L, _ = gather_factor(an.symbol, res.store)
    assert rel(L, np.linalg.cholesky(an.A_perm.to_dense())) <= 1e-12


def test_indefinite_raises_reference_column():
    A = sparse.shift_diagonal(sparse.gen_laplacian(3, (6, 6, 6)), 2.0)
    an = analyze(A)
    with pytest.raises(NotPositiveDefiniteError) as eo:
        O.factor_analysis(an)
    with pytest.raises(NotPositiveDefiniteError) as eg:
        factorize(an)
    assert eg.value.column == eo.value.column
    assert abs(eg.value.pivot - eo.value.pivot) <= 1e-10 * max(1.0, abs(eo.value.pivot))


def test_ldlt_singular_pivot_raises():
    # exact zero pivot: diag(1, 0) with no coupling
    A = sparse.from_coo(2, [0, 1], [0, 1], [1.0, 0.0], "symmetric-lower")
    an = analyze(A, AnalyzeOptions(form="ldlt"))
    with pytest.raises(SingularPivotError) as e:
        factorize(an)
    assert e.value.column == an.perm.perm[1]


def test_deterministic_bitwise():
    A = sparse.gen_laplacian(3, (16, 16, 16))
    an = analyze(A)
    a = factorize(an).store.slab.copy()
    b = factorize(an).store.slab.copy()
    assert np.array_equal(a, b)


def test_host_store_survives_next_factorization():
    """The pinned host slab is recycled only when nothing references it."""
    an = analyze(sparse.gen_laplacian(3, (10, 10, 10)))
    first = factorize(an).store          # keep the PanelStore, drop the result
    snap = first.slab.copy()
    for _ in range(3):
        factorize(an).store.slab[:] = -1.0   # results dropped -> buffers recycled
    assert np.array_equal(first.slab, snap)


@pytest.mark.parametrize("form,shift", [("llt", 0.0), ("ldlt", 0.5)])
def test_overlapped_download_equals_device_slab(form, shift):
    """factorize(download=True) moves the slab chunk by chunk while the factor
    runs (ps_factor_download): the host slab must equal the device slab
    bitwise, and equal the factor of the non-overlapped path."""
    A = sparse.gen_laplacian(3, (20, 20, 20))
    if shift:
        A = sparse.shift_diagonal(A, shift)
    an = analyze(A, AnalyzeOptions(form=form))
    r1 = factorize(an, download=True)
    host = r1.store.slab.copy()
    dev = r1.device_store.tensor.cpu().numpy()
    assert np.array_equal(host, dev)
    r2 = factorize(an, download=False)
    assert np.array_equal(r2.store.slab, host)
    for _ in range(2):  # pooled slabs reused: still exact
        assert np.array_equal(factorize(an).store.slab, host)


@pytest.mark.parametrize("N", [40])
def test_factorize_lap3d_oracle(N):
    A = sparse.gen_laplacian(3, (N, N, N))
    an = analyze(A)
    res = factorize(an)
    ref = O.factor_analysis(an)
    assert rel(res.store.slab, ref.slab) <= 1e-12


@pytest.mark.parametrize("form,nranks", [("llt", 2), ("ldlt", 2), ("llt", 4)])
def test_partitioned_rank_plans_on_one_gpu(form, nranks):
    """Every rank's plan (phase 0: own subtrees + fan-in contributions into
    its top copy), the top-region sum (what NCCL reduce does across GPUs),
    then phase 1 on rank 0 == the single-GPU factor."""
    from paper_1405_2636_b200.distributed import (check_partition, entry_owner_mask,
                                                  partition, top_range)
    from paper_1405_2636_b200.pipeline import default_pivot_threshold
    from paper_1405_2636_b200.symbolic import assembly_positions
    A = sparse.gen_laplacian(3, (16, 16, 16))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    an = analyze(A, AnalyzeOptions(form=form))
    sym = an.symbol
    group = partition(sym, nranks, form)
    check_partition(sym, group)
    lo, hi = top_range(sym, group)
    thr = default_pivot_threshold(an.A_perm)
    pos, sel = assembly_positions(sym, an.A_perm)
    stores, engines = [], []
    for r in range(nranks):
        eng = Engine(sym, "cuda:0", partition=(group, nranks, r))
        st = eng.new_store()
        mine = entry_owner_mask(sym, an.A_perm, group, r)
        eng.assemble_positions(st, torch.from_numpy(pos[mine]).cuda(),
                               torch.from_numpy(np.ascontiguousarray(an.A_perm.values[sel][mine])).cuda())
        eng.factor(st, form, thr, phase=0)
        eng.check(form)
        stores.append(st)
        engines.append(eng)
    full = stores[0]
    for r in range(1, nranks):
        full += stores[r]          # owned regions are disjoint; the top sums the fan-in
    engines[0].factor(full, form, thr, phase=1)
    engines[0].check(form)
    ref = factorize(an).store.slab
    # LLt on an SPD Laplacian is order-insensitive (<= 1.8e-16);
    # the shifted indefinite LDLt is not (the reference disagrees with itself
    # by 3.0e-11 at 24^3), so the partitioned summation order gets the
    # north-star factor tolerance
    tol = 1e-12 if form == "llt" else 1e-11
    err = rel(full.cpu().numpy(), ref)
    print(f"partitioned vs single-GPU factor ({form}): {err:.2e}")
    assert err <= tol


# --------------------------------------------------------------------------
# GPU supernodal solve (ps_solve) vs the host restatement of supernodal_solve

@pytest.mark.parametrize("dims,form,shift", [((16, 16), "llt", 0.0), ((10, 10, 10), "llt", 0.0),
                                            ((10, 10, 10), "ldlt", 0.5), ((24, 24, 24), "llt", 0.0),
                                            ((12, 12, 12), "ldlt", 0.5)])
def test_gpu_solve_vs_host(dims, form, shift):
    from paper_1405_2636_b200.solve import supernodal_solve
    A = sparse.gen_laplacian(len(dims), dims)
    if shift:
        A = sparse.shift_diagonal(A, shift)
    an = analyze(A, AnalyzeOptions(form=form))
    res = factorize(an)
    rng = np.random.default_rng(7)
    b = rng.standard_normal(A.n)
    xg = res.solve(b)
    xh = supernodal_solve(an.symbol, res.store, b, form, an.perm.perm)
    assert np.abs(xg - xh).max() <= 1e-10 * np.abs(xh).max()
    bb = sparse.spmv(A, np.ones(A.n))
    assert sparse.backward_error(A, res.solve(bb, refine=1), bb) <= 1e-12


@pytest.mark.parametrize("smem_w", ["4096", "0"])
def test_gpu_solve_wide_panel(smem_w, monkeypatch):
    """A dense 300-wide panel; smem_w=0 forces the global-scratch path used by
    panels wider than the shared-memory right-hand side (120^3: w = 12578)."""
    from paper_1405_2636_b200.solve import supernodal_solve
    monkeypatch.setenv("PS_SOLVE_SMEM_W", smem_w)
    rng = np.random.default_rng(3)
    n = 300
    M = rng.standard_normal((n, n))
    D = M @ M.T + n * np.eye(n)
    r, c = np.tril_indices(n)
    A = sparse.from_coo(n, r, c, D[r, c], "symmetric-lower")
    an = analyze(A)
    res = factorize(an)
    b = rng.standard_normal(n)
    xg = res.solve(b)
    assert np.abs(D @ xg - b).max() <= 1e-10 * np.abs(b).max()
    xh = supernodal_solve(an.symbol, res.store, b, "llt", an.perm.perm)
    assert np.abs(xg - xh).max() <= 1e-10 * np.abs(xh).max()
