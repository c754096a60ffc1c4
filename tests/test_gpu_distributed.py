"""The multi-process factorization path end to end on the GPU box: torchrun
with 2 ranks over gloo sharing cuda:0 (the pool gives one GPU; production is
NCCL with one GPU per rank).  Rank plans, fan-in reduce of the top region and
the top factorization must reproduce the single-GPU factor."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,N,form,port,dtop", [(2, 16, "llt", 29611, "0"),
                                                    (2, 14, "ldlt", 29612, "0"),
                                                    (3, 16, "llt", 29613, "0"),
                                                    (2, 16, "llt", 29614, "1"),
                                                    (3, 18, "llt", 29615, "1"),
                                                    (2, 14, "ldlt", 29616, "1")])
def test_two_rank_factorization_matches_single_gpu(world, N, form, port, dtop):
    """dtop=1: top separators distributed over the ranks (owners factor,
    broadcast per top level, owners of destinations apply the updates)."""
    env = dict(os.environ, PS_DIST_BACKEND="gloo", PS_DIST_SAME_DEVICE="1", PS_DIST_TOP=dtop)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tools", "dist_check.py"), str(N), form]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "OK" in r.stdout
