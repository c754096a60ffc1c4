"""Factor parity with the REFERENCE at the BASELINE configurations.

Fixtures tests/golden/big_<case>.npz hold a strided sample and 8192 chunk
norms of the reference's own factor slab (tests/golden/make_golden_big.py
ran the reference: sequential scheduler, 1 BLAS thread; for the shifted
LDLt case also its dynamic scheduler, whose schedule-to-schedule spread sets
the tolerance).  The engine's slab has the reference's
PanelStore layout, so entries are compared position for position on the
device (no download of the factor).

Tolerances (north star: factor entries within 1e-10 relative, backward error
<= 1e-12):
  LLt           max|dL| / max|L| <= 1e-10 on the sample; chunk norms <= 1e-10
                relative; raw ||Ax-b||/||b|| <= 1e-12
  shifted LDLt  max|dL| / max|L| <= 10x the reference's own spread; chunk
                norms <= 10x its chunk spread; ||Ax-b||/||b|| <= 1e-12 after
                one refinement step (the reference itself reaches 1.1e-10 raw)
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.pipeline import factorize  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NCHUNK = 8192


def load(case):
    path = os.path.join(GOLDEN, f"big_{case}.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {path} not generated")
    return dict(np.load(path))


def chunk_norms_dev(t):
    n = t.numel()
    edges = np.linspace(0, n, NCHUNK + 1).astype(np.int64)
    out = np.empty(NCHUNK)
    for c in range(NCHUNK):
        out[c] = float(torch.linalg.vector_norm(t[edges[c]:edges[c + 1]]))
    return out


def run_case(case, slow_ok=True):
    g = load(case)
    N, shift, form = int(g["N"]), float(g["shift"]), str(g["form"])
    A = sparse.gen_laplacian(3, (N, N, N))
    if shift:
        A = sparse.shift_diagonal(A, shift)
    an = analyze(A, AnalyzeOptions(form=form))
    assert an.flops == int(g["flops"])
    res = factorize(an, download=False)
    t = res.device_store.tensor
    assert t.numel() == int(g["size"])
    stride = int(g["stride"])
    sample = t[::stride].cpu().numpy()
    err = float(np.abs(sample - g["sample"]).max() / g["max_abs"])
    cn = chunk_norms_dev(t)
    cerr = float(np.max(np.abs(cn - g["chunk_norm"]) / np.maximum(g["chunk_norm"], 1e-300)))
    b = sparse.spmv(A, np.ones(A.n))
    x = res.solve(b)
    berr = sparse.backward_error(A, x, b)
    x1 = res.solve(b, refine=1)
    berr1 = sparse.backward_error(A, x1, b)
    return g, err, cerr, berr, berr1


def test_lap3d_40_llt_vs_reference():
    g, err, cerr, berr, berr1 = run_case("lap3d_40_llt")
    assert err <= 1e-10 and cerr <= 1e-10, (err, cerr)
    assert berr <= 1e-12, berr


def test_lap3d_60_llt_vs_reference():
    # C2: the bench configuration of round 1
    g, err, cerr, berr, berr1 = run_case("lap3d_60_llt")
    assert err <= 1e-10 and cerr <= 1e-10, (err, cerr)
    assert berr <= 1e-12, berr


def test_lap3d_80_ldlt_shift_vs_reference():
    # C3: symmetric indefinite A - 0.5 I
    g, err, cerr, berr, berr1 = run_case("lap3d_80_ldlt_shift")
    assert err <= 10 * float(g["spread"]), (err, float(g["spread"]))
    assert cerr <= 10 * float(g["spread_chunk"]), (cerr, float(g["spread_chunk"]))
    assert berr <= 10 * float(g["berr"]), (berr, float(g["berr"]))
    assert berr1 <= 1e-12, berr1


@pytest.mark.slow
def test_lap3d_120_llt_vs_reference():
    # C5 at one GPU: the north-star configuration
    g, err, cerr, berr, berr1 = run_case("lap3d_120_llt")
    assert err <= 1e-10 and cerr <= 1e-10, (err, cerr)
    assert berr <= 1e-12, berr
