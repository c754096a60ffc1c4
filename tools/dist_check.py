"""Multi-process factorization check (launched by torchrun).

Every rank runs DistributedFactorizer (subtree partition, fan-in reduce of the
top region, top on rank 0); rank 0 compares the gathered factor with the
single-GPU factor and the backward error.  PS_DIST_BACKEND=gloo with
PS_DIST_SAME_DEVICE=1 lets several ranks share one GPU (CI on a 1-GPU box);
the production path is NCCL, one GPU per rank.
  torchrun --nproc-per-node G tools/dist_check.py N form"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.distributed import DistributedFactorizer
from paper_1405_2636_b200.pipeline import factorize, DeviceStore
from paper_1405_2636_b200.solve import supernodal_solve

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
backend = os.environ.get("PS_DIST_BACKEND", "nccl")
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0"))
dev = torch.device("cuda", 0 if os.environ.get("PS_DIST_SAME_DEVICE") else local)
torch.cuda.set_device(dev)
dist.init_process_group(backend)
A = sparse.gen_laplacian(3, (N, N, N))
if form == "ldlt":
    A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
dtop = os.environ.get("PS_DIST_TOP", "0") == "1"
dfz = DistributedFactorizer(an, rank, world, dev, distribute_top=dtop)
dfz.assemble()
dfz.factor()
if dtop:
    dfz.check()
elif rank == 0:
    dfz.check()
full = dfz.gather_factor_slab()
ok = True
if rank == 0:
    ref = factorize(an, device=dev).store.slab
    got = full.cpu().numpy()
    err = float(np.abs(got - ref).max() / np.abs(ref).max())
    hs = DeviceStore(an.symbol, full).to_host()
    b = sparse.spmv(A, np.ones(A.n))
    berr = sparse.backward_error(A, supernodal_solve(an.symbol, hs, b, form, an.perm.perm), b)
    tol = 1e-12 if form == "llt" else 1e-10
    ok = err <= tol and berr <= (1e-12 if form == "llt" else 1e-8)
    top = int((dfz.group < 0).sum())
    print(f"world {world} {backend} distribute_top={dtop}: factor rel err vs 1-GPU {err:.2e}, backward error {berr:.2e}, "
          f"top panels {top} of {an.symbol.npanels}: {'OK' if ok else 'FAIL'}", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
