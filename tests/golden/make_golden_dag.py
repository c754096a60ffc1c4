"""Reference task DAGs (export_dag text + priorities) for small cases.

Build container only (imports the reference from /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dag.py
Writes tests/golden/dag_<case>.txt (taskgraph.py:141-153 format) followed by
a `priorities` section (taskgraph.py:123-138).
"""

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(__file__))
from panelsolve import pipeline, sparse, taskgraph  # noqa: E402  (the reference)
from make_golden import shifted  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    yield "lap2d_16_llt", sparse.gen_laplacian(2, (16, 16)), "llt"
    yield "lap3d_8_ldlt_shift", shifted(sparse.gen_laplacian(3, (8, 8, 8)), 0.5), "ldlt"


for name, A, form in cases():
    an = pipeline.analyze(A, pipeline.AnalyzeOptions(form=form))
    path = os.path.join(HERE, f"dag_{name}.txt")
    taskgraph.export_dag(an.graph, path)
    with open(path, "a") as fh:
        fh.write(f"priorities {len(an.graph.tasks)}\n")
        for t in an.graph.tasks:
            fh.write(f"{t.id} {t.priority}\n")
    print(name, len(an.graph.tasks), an.graph.nedges)
