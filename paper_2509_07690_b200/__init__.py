"""B200-native HYLU numeric factorization, refactorization and solve.

Drop-in for the reference package's (``polylu``) analyze / factorize /
refactorize / solve surface; see ``api.py`` for the SPEC mapping and DESIGN.md
for the device design.
"""

from ._ref import KernelMode, SolverConfig, SparseMatrixCSR, errors  # noqa: F401
from .analysis import Analysis, analyze  # noqa: F401
from .api import (  # noqa: F401
    BatchedRefactorizer,
    FactorOptions,
    NumericFactors,
    Ordering,
    PivotScale,
    RefinementReport,
    amd_order,
    factorize,
    factorize_analysis,
    refactorize,
    refactorize_solve_batched,
    solve,
    static_pivot,
    substitute,
    symbolic_factorize,
)
from .symbolic import SymbolicStructure, select_kernel  # noqa: F401

__version__ = "0.1.0"
