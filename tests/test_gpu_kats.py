"""The reference's kernel known-answer tests (pkg/tests/test_kernels.py:22-83,
200-241) run through the CUDA factor operator `ps_run_factor_task` (one
factor task = diagonal factor + panel TRSM, kernels.py:208-247) instead of
the stand-alone numpy kernels."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1405_2636_b200.engine import Engine  # noqa: E402
from paper_1405_2636_b200.errors import NotPositiveDefiniteError, SingularPivotError  # noqa: E402
from paper_1405_2636_b200.symbolic import PanelSet, PanelStore, build_symbol  # noqa: E402


def one_panel(block, rows=None):
    """Panel 0 = the dense lower block (w x w) plus off-diagonal rows `rows`
    (each of length w), facing a second panel when rows are given."""
    block = np.asarray(block, dtype=np.float64)
    w = block.shape[0]
    rows = np.zeros((0, w)) if rows is None else np.asarray(rows, dtype=np.float64)
    m = rows.shape[0]
    if m:
        ps_ = PanelSet(np.array([0, w, w + m]), [np.arange(w, w + m, dtype=np.int64),
                                                 np.zeros(0, dtype=np.int64)])
    else:
        ps_ = PanelSet(np.array([0, w]), [np.zeros(0, dtype=np.int64)])
    sym = build_symbol(ps_)
    host = PanelStore(sym)
    a = host.data[0]
    a[:w, :] = np.tril(block)
    a[w:, :] = rows
    return sym, host


def run(block, rows=None, form="llt", thr=0.0, upper=None):
    sym, host = one_panel(block, rows)
    if upper is not None:
        w = host.data[0].shape[1]
        host.data[0][np.triu_indices(w, 1)] = upper
    eng = Engine(sym)
    dev = torch.from_numpy(host.slab.copy()).cuda()
    eng.run_factor_task(dev, 0, form, thr)
    return PanelStore(sym, slab=dev.cpu().numpy()).data[0]


def test_potrf_identity():
    assert np.array_equal(run(np.eye(2)), np.eye(2))


def test_potrf_two_by_two():
    # test_kernels.py:29-33: [[4,2],[2,3]] -> [[2,0],[1,sqrt 2]]
    a = run([[4.0, 0.0], [2.0, 3.0]])
    assert a[0, 0] == 2.0 and a[1, 0] == 1.0 and abs(a[1, 1] - np.sqrt(2)) <= 1e-15
    assert a[0, 1] == 0.0


def test_potrf_indefinite_names_column():
    # test_kernels.py:35-39
    with pytest.raises(NotPositiveDefiniteError) as err:
        run([[1.0, 0.0], [2.0, 1.0]])
    assert err.value.column == 1


@pytest.mark.parametrize("w", [6, 33, 70])
def test_potrf_upper_triangle_untouched(w):
    # test_kernels.py:41-47: a canary in the strict upper triangle survives
    rng = np.random.default_rng(20240211 + w)
    M = rng.uniform(-1, 1, (w, w))
    Ad = M + M.T + np.diag(2 * w * np.ones(w))
    a = run(Ad, upper=123.456)
    assert np.all(a[np.triu_indices(w, 1)] == 123.456)
    assert np.abs(np.tril(a) - np.linalg.cholesky(Ad)).max() <= 1e-13 * np.abs(a).max()


def test_trsm_scalar():
    # test_kernels.py:66-70: L = [[2]], B = [[6],[8]] -> [[3],[4]]
    a = run([[4.0]], rows=[[6.0], [8.0]])
    assert a[:, 0].tolist() == [2.0, 3.0, 4.0]


def test_trsm_identity_diag():
    # test_kernels.py:59-64
    B = np.arange(6, dtype=float).reshape(2, 3)
    a = run(np.eye(3), rows=B)
    assert np.array_equal(a[3:], B)


def test_ldlt_already_diagonal():
    # test_kernels.py:201-205
    a = run(np.diag([2.0, -3.0]), form="ldlt")
    assert np.diagonal(a).tolist() == [2.0, -3.0] and a[1, 0] == 0.0


def test_ldlt_two_by_two():
    # test_kernels.py:207-211: [[2,2],[2,5]] -> L10 = 1, d = (2, 3)
    a = run([[2.0, 0.0], [2.0, 5.0]], form="ldlt")
    assert a[1, 0] == 1.0 and np.diagonal(a).tolist() == [2.0, 3.0]


def test_ldlt_singular_pivot():
    # test_kernels.py:213-217
    with pytest.raises(SingularPivotError) as err:
        run([[0.0]], form="ldlt", thr=1e-13)
    assert err.value.column == 0


def test_ldlt_trsm():
    # test_kernels.py:219-225: x (D L^T) = [4, 10] -> [2, 2]
    a = run([[2.0, 0.0], [2.0, 5.0]], rows=[[4.0, 10.0]], form="ldlt")
    assert np.abs(a[2] - np.array([2.0, 2.0])).max() <= 1e-14
