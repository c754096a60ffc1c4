"""Device task runtime (ps_dataflow.cuh, PS_SCHED=dataflow): the whole
factorization as one persistent kernel over the refined task DAG of the
reference (taskgraph.py:79-110).  Parity with the oracle and with the level
schedule, bitwise determinism, the reference's error semantics, and a
consistent exported task graph."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import panel_oracle as O  # noqa: E402
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.engine import Engine  # noqa: E402
from paper_1405_2636_b200.errors import NotPositiveDefiniteError, SingularPivotError  # noqa: E402,F401
from paper_1405_2636_b200.pipeline import default_pivot_threshold  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dataflow_engine(sym):
    old = os.environ.get("PS_SCHED")
    os.environ["PS_SCHED"] = "dataflow"
    try:
        eng = Engine(sym, "cuda:0")
    finally:
        if old is None:
            del os.environ["PS_SCHED"]
        else:
            os.environ["PS_SCHED"] = old
    assert eng.dataflow_info()["built"] == 1
    return eng


def run(eng, an, form, sched):
    eng.set_schedule(sched)
    st = eng.new_store()
    eng.assemble(st, an.A_perm)
    eng.factor(st, form, default_pivot_threshold(an.A_perm))
    eng.check(form)
    return st.cpu().numpy()


@pytest.mark.parametrize("dims,form,shift", [((16, 16), "llt", 0.0), ((8, 8, 8), "llt", 0.0),
                                            ((8, 8, 8), "ldlt", 0.5), ((16, 16, 16), "llt", 0.0),
                                            ((24, 24, 24), "llt", 0.0), ((16, 16, 16), "ldlt", 0.5)])
def test_dataflow_vs_oracle_and_level(dims, form, shift):
    A = sparse.gen_laplacian(len(dims), dims)
    if shift:
        A = sparse.shift_diagonal(A, shift)
    an = analyze(A, AnalyzeOptions(form=form))
    eng = dataflow_engine(an.symbol)
    df = run(eng, an, form, "dataflow")
    lv = run(eng, an, form, "level")
    ref = O.factor_analysis(an).slab
    tol = 1e-12 if form == "llt" else 1e-10  # shifted LDLt: order-sensitive
    assert rel(df, ref) <= tol
    assert rel(df, lv) <= tol


def test_dataflow_bitwise_deterministic():
    an = analyze(sparse.gen_laplacian(3, (20, 20, 20)), AnalyzeOptions())
    eng = dataflow_engine(an.symbol)
    a = run(eng, an, "llt", "dataflow")
    b = run(eng, an, "llt", "dataflow")
    assert np.array_equal(a, b)


def test_dataflow_indefinite_raises_reference_column():
    A = sparse.shift_diagonal(sparse.gen_laplacian(3, (6, 6, 6)), 2.0)
    an = analyze(A, AnalyzeOptions())
    with pytest.raises(NotPositiveDefiniteError) as eo:
        O.factor_analysis(an)
    eng = dataflow_engine(an.symbol)
    eng.set_schedule("dataflow")
    st = eng.new_store()
    eng.assemble(st, an.A_perm)
    eng.factor(st, "llt", default_pivot_threshold(an.A_perm))
    with pytest.raises(NotPositiveDefiniteError) as eg:
        eng.check("llt")
    assert eg.value.column == eo.value.column
    assert abs(eg.value.pivot - eo.value.pivot) <= 1e-10 * max(1.0, abs(eo.value.pivot))


def test_dataflow_ldlt_singular_pivot_raises():
    A = sparse.from_coo(2, [0, 1], [0, 1], [1.0, 0.0], "symmetric-lower")
    an = analyze(A, AnalyzeOptions(form="ldlt"))
    eng = dataflow_engine(an.symbol)
    eng.set_schedule("dataflow")
    st = eng.new_store()
    eng.assemble(st, an.A_perm)
    eng.factor(st, "ldlt", default_pivot_threshold(an.A_perm))
    with pytest.raises(SingularPivotError) as e:
        eng.check("ldlt")
    assert e.value.column == an.perm.perm[1]


def test_dataflow_task_graph_is_consistent():
    """Every dependency threshold is reachable: the signal count of each
    counter covers the largest target waiting on it; the trace covers every
    task once."""
    an = analyze(sparse.gen_laplacian(3, (12, 12, 12)), AnalyzeOptions())
    eng = dataflow_engine(an.symbol)
    dep_ptr, dep_ctr, dep_tg, sig_ptr, sig_ctr = eng.task_graph()
    n = int(eng.dataflow_info()["ntasks"])
    assert len(dep_ptr) == n + 1 and len(sig_ptr) == n + 1
    counts = np.bincount(sig_ctr, minlength=int(dep_ctr.max()) + 1 if len(dep_ctr) else 1)
    for c, t in zip(dep_ctr, dep_tg):
        assert counts[c] >= t
    st = eng.new_store()
    eng.assemble(st, an.A_perm)
    tr = eng.factor_trace(st, "llt", default_pivot_threshold(an.A_perm))
    eng.check("llt")
    assert (tr[:, 1] > 0).all() and (tr[:, 3] >= tr[:, 1]).all()
