"""Drop-in boundary details: traces in the reference schema, one plan per
device, the reference's per-call pivot threshold, host registration."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.errors import NotPositiveDefiniteError  # noqa: E402
from paper_1405_2636_b200.pipeline import check_solve, factorize  # noqa: E402
from paper_1405_2636_b200.taskgraph import FACTOR, UPDATE  # noqa: E402
from paper_1405_2636_b200.trace import read_trace_csv, trace_to_csv  # noqa: E402


def test_trace_covers_every_task_once(tmp_path):
    # reference runtime.py:314-317: the trace covers every task exactly once
    A = sparse.gen_laplacian(3, (12, 12, 12))
    an = analyze(A)
    res = factorize(an, collect_trace=True)
    ev = res.events
    g = an.graph
    assert sorted(e.task_id for e in ev) == list(range(len(g.tasks)))
    for e in ev:
        t = g.tasks[e.task_id]
        assert (e.kind, e.p, e.q) == (t.kind, t.p, t.q)
        assert 0 <= e.start_ns <= e.end_ns
    # dependencies: an update ends no earlier than its source factor starts
    start = {e.task_id: e.start_ns for e in ev}
    end = {e.task_id: e.end_ns for e in ev}
    for (p, q), u in g.update_of.items():
        assert end[u] >= start[p]
        assert start[q] <= end[q]
    path = tmp_path / "trace.csv"
    trace_to_csv(ev, path)
    assert open(path).readline().strip() == "task_id,kind,src,dst,worker,start_ns,end_ns"
    back = read_trace_csv(path)
    assert sorted(back, key=lambda e: e.task_id) == sorted(ev, key=lambda e: e.task_id)
    assert {e.kind for e in ev} == {FACTOR, UPDATE}
    # the replay did not touch the result
    r, _ = check_solve(A, res)
    assert r <= 1e-12


def test_no_trace_when_not_collected():
    an = analyze(sparse.gen_laplacian(2, (16, 16)))
    assert factorize(an, collect_trace=False).events == []


def test_one_plan_per_device():
    A = sparse.gen_laplacian(2, (20, 20))
    an = analyze(A)
    r1 = factorize(an)
    r1.solve(np.ones(A.n))
    r2 = factorize(an, device="cuda:0")
    r3 = factorize(an, device=torch.device("cuda", 0))
    r3.solve(np.ones(A.n))
    assert len(an._engines) == 1
    assert np.array_equal(r1.store.slab, r2.store.slab)
    # torch's CUDA error state stays clean (registration goes through the engine)
    x = torch.zeros(4, device="cuda")
    x[torch.tensor([1, 2], device="cuda")] = 1.0
    torch.cuda.synchronize()


def test_threshold_recomputed_per_call():
    # reference pipeline.py:88-91: default_pivot_threshold(A_perm) on every call
    A = sparse.gen_laplacian(3, (6, 6, 6))
    an = analyze(A)
    factorize(an)
    on = an.A_perm.rowidx == an.A_perm.entry_cols()
    an.A_perm.values[on] -= 2.0  # in place: now indefinite
    with pytest.raises(NotPositiveDefiniteError):
        factorize(an)


def test_device_default_threshold_boundary():
    # factorize() hands the engine a NaN threshold: the reference default
    # 1e-13 max|diag(A)| (kernels.py:32-40) is computed on the device from the
    # assembled slab.  Column 0 decoupled, its pivot just below / above it:
    # LLt fails there iff piv <= thr (kernels.py:217-221).
    A = sparse.gen_laplacian(3, (6, 6, 6))
    an = analyze(A)
    P = an.A_perm
    c0, c1 = P.colptr[0], P.colptr[1]
    rows = P.rowidx[c0:c1]
    off = [k for k in range(c0, c1) if P.rowidx[k] != 0]
    diag = c0 + int(np.flatnonzero(rows == 0)[0])
    P.values[off] = 0.0
    m = float(np.abs(P.values[P.rowidx == P.entry_cols()]).max())
    P.values[diag] = 0.5e-13 * m
    with pytest.raises(NotPositiveDefiniteError) as ei:
        factorize(an)
    assert ei.value.column == 0
    P.values[diag] = 2e-13 * m
    factorize(an)  # above the threshold: no failure


def test_device_default_threshold_boundary_complex_lu():
    # the device threshold on complex128 slabs (|x| = hypot) and the LU
    # failure predicate |piv| <= thr: column 0 decoupled (its row and column),
    # its pivot just below / above 1e-13 max|diag(A)|
    from paper_1405_2636_b200.errors import SingularPivotError
    A = sparse.gen_convdiff27(5, complex_shift=1.0)
    an = analyze(A, AnalyzeOptions(form="lu"))
    P = an.A_perm
    cols = P.entry_cols()
    P.values[((cols == 0) & (P.rowidx != 0)) | ((P.rowidx == 0) & (cols != 0))] = 0.0
    d0 = int(np.flatnonzero((cols == 0) & (P.rowidx == 0))[0])
    m = float(np.abs(P.values[P.rowidx == cols]).max())
    P.values[d0] = 0.5e-13 * m * (0.6 + 0.8j)
    with pytest.raises(SingularPivotError) as ei:
        factorize(an)
    assert ei.value.column == 0
    P.values[d0] = 2e-13 * m * (0.6 + 0.8j)
    factorize(an)
