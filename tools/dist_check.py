"""Multi-process factorization check (launched by torchrun).

Every rank runs DistributedFactorizer (subtree partition, fan-in of the top,
the top on rank 0 or distributed over owners; PS_DIST_TRANSPORT=p2p|nccl)
twice; rank 0 compares the gathered factor with the oracle (the checker),
checks the two factorizations are bitwise equal and the backward error
(LDLt: after one refinement step).  PS_DIST_BACKEND=gloo with
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
transport = os.environ.get("PS_DIST_TRANSPORT", "p2p")
dfz = DistributedFactorizer(an, rank, world, dev, distribute_top=dtop, transport=transport)
slabs = []
for it in range(2):  # two factorizations: the p2p epoch protocol across calls
    dfz.assemble()
    dfz.factor()
    if dtop:
        dfz.check()
    elif rank == 0:
        dfz.check()
    full = dfz.gather_factor_slab()
    if rank == 0:
        slabs.append(full.cpu().numpy())
ok = True
if rank == 0:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import panel_oracle as O  # test infrastructure: the checker
    ref = O.factor_analysis(an).slab
    got = slabs[-1]
    err = float(np.abs(got - ref).max() / np.abs(ref).max())
    same = bool(np.array_equal(slabs[0], slabs[1]))
    hs = DeviceStore(an.symbol, full).to_host()
    b = sparse.spmv(A, np.ones(A.n))
    x = supernodal_solve(an.symbol, hs, b, form, an.perm.perm)
    berr = sparse.backward_error(A, x, b)
    x1 = x + supernodal_solve(an.symbol, hs, b - sparse.spmv(A, x), form, an.perm.perm)
    berr1 = sparse.backward_error(A, x1, b)
    tol = 1e-12 if form == "llt" else 1e-10
    ok = err <= tol and same and (berr if form == "llt" else berr1) <= 1e-12
    top = int((dfz.group < 0).sum())
    print(f"world {world} {backend} distribute_top={dtop} transport={dfz.transport}: factor rel err "
          f"vs oracle {err:.2e}, repeat bitwise {same}, backward error {berr:.2e} "
          f"(1 refinement step {berr1:.2e}), top panels {top} of {an.symbol.npanels}: "
          f"{'OK' if ok else 'FAIL'}", flush=True)
dfz.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
