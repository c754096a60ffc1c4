"""Analysis.graph / export_dag restate the reference's task DAG
(taskgraph.py:79-153): identical text export and priorities on the DAGs the
reference itself wrote (tests/golden/make_golden_dag.py)."""

import os

import pytest

from _cases import small_case
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
from paper_1405_2636_b200.taskgraph import FACTOR, UPDATE, export_dag

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["lap2d_16_llt", "lap3d_8_ldlt_shift"])
def test_dag_equals_reference(name, tmp_path):
    A, form = small_case(name)
    an = analyze(A, AnalyzeOptions(form=form))
    g = an.graph
    out = tmp_path / "dag.txt"
    export_dag(g, out)
    with open(out, "a") as fh:
        fh.write(f"priorities {len(g.tasks)}\n")
        for t in g.tasks:
            fh.write(f"{t.id} {t.priority}\n")
    assert out.read_text() == open(os.path.join(GOLDEN, f"dag_{name}.txt")).read()


def test_dag_structure():
    A, form = small_case("lap2d_16_llt")
    an = analyze(A, AnalyzeOptions(form=form))
    g = an.graph
    assert len(g) == an.symbol.npanels + len(g.update_of)
    order = g.topological_order()
    pos = {t: i for i, t in enumerate(order)}
    for t in g.tasks:
        for s in t.successors:
            assert pos[t.id] < pos[s]
        if t.kind == FACTOR:
            assert all(g.tasks[s].kind == UPDATE and g.tasks[s].p == t.p for s in t.successors)
    assert sum(t.cost for t in g.tasks) == an.flops
