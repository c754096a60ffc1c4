"""The multi-process factorization path end to end on the GPU box: torchrun
with 2-4 ranks sharing cuda:0 (the pool gives one GPU; production is one GPU
per rank over NVLink).  Rank plans, the fan-in of the top and the top
factorization must reproduce the oracle's factor (LLt <= 1e-12, shifted LDLt
<= 1e-10 relative), bitwise repeatably, with backward error <= 1e-12."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,N,form,port,dtop,transport", [
    (2, 16, "llt", 29611, "0", "nccl"),
    (2, 14, "ldlt", 29612, "0", "nccl"),
    (3, 16, "llt", 29613, "0", "nccl"),
    (2, 16, "llt", 29614, "1", "nccl"),
    (3, 18, "llt", 29615, "1", "nccl"),
    (2, 16, "llt", 29616, "1", "p2p"),
    (3, 18, "llt", 29617, "1", "p2p"),
    (4, 18, "llt", 29618, "1", "p2p"),
    (2, 14, "ldlt", 29619, "1", "p2p")])
def test_multi_rank_factorization_matches_oracle(world, N, form, port, dtop, transport):
    """dtop=1: top separators distributed over the ranks (owners factor, the
    factored panels reach the owners of their destinations - NCCL broadcasts
    or peer pulls through CUDA IPC - and those apply the updates)."""
    env = dict(os.environ, PS_DIST_BACKEND="gloo", PS_DIST_SAME_DEVICE="1", PS_DIST_TOP=dtop,
               PS_DIST_TRANSPORT=transport)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tools", "dist_check.py"), str(N), form]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "OK" in r.stdout
