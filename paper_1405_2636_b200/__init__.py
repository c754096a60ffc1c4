"""B200-native numeric factorization for the supernodal sparse direct solver
of arXiv 1405.2636 (drop-in for the reference `panelsolve` numeric path).

    an  = analyze(A, AnalyzeOptions(form="llt"))      # host: ordering + symbol
    res = factorize(an)                               # sm_100a CUDA engine
    x   = res.solve(b)
"""

from .analysis import Analysis, AnalyzeOptions, analyze
from .errors import (DeviceError, DivergentSolveError,
                     NotPositiveDefiniteError, SingularPivotError, StructuralError)
from .flops import LDLT, LLT, total_flops
from .pipeline import (FactorResult, check_solve, default_pivot_threshold, factorize,
                       run_report)
from .solve import supernodal_solve
from .sparse import (SparseMatrix, backward_error, gen_convdiff27, gen_laplacian,
                     residual_norm, shift_diagonal, spmv, symmetrize_pattern)
from .symbolic import allocate_panels, gather_factor

__version__ = "0.1.0"

__all__ = [
    "Analysis", "AnalyzeOptions", "DeviceError", "DivergentSolveError", "FactorResult",
    "LDLT", "LLT", "NotPositiveDefiniteError", "SingularPivotError",
    "SparseMatrix", "StructuralError", "allocate_panels", "analyze", "check_solve",
    "default_pivot_threshold", "factorize", "gather_factor", "gen_convdiff27",
    "gen_laplacian", "backward_error", "residual_norm", "run_report", "shift_diagonal",
    "spmv", "supernodal_solve", "symmetrize_pattern", "total_flops",
]
