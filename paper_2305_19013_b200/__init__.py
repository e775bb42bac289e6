"""B200-native hot loop of the memory-reduced enlarged CG family (arXiv 2305.19013).

Drop-in for the reference `ekcg` solver path: same `enlarged_solve`,
`SolverConfig`, `ConvergenceReport`, `SparseSpdMatrix`, `Partition` and
per-kernel functions, executed by hand-written sm_100a fp64 kernels
(libekcg_b200.so, C ABI in include/ekcg_b200.h).
"""

from .linalg import (
    Breakdown,
    SparseSpdMatrix,
    cholesky_small,
    gram,
    norm2,
    spmm,
    spmv,
    trsm_right_inv,
)
from .partition import Partition, contiguous_partition, read_partition, write_partition
from .aortho import a_cholqr, a_orthogonalize_against, pre_cholqr
from .cg import cg
from .operators import CsrOperator, StencilOperator, as_operator
from .solvers import (
    METHODS,
    RETENTIONS,
    BasisStore,
    ConvergenceReport,
    SolverConfig,
    enlarged_solve,
)
from .precond import (
    BlockJacobiFactor,
    aligned_with,
    apply_minv,
    backward_solve,
    build_block_jacobi,
    forward_solve,
    uniform_block_bounds,
)
from .reporting import CSV_COLUMNS, make_rhs, run_batch, run_experiment, write_history, write_runs_csv
from .problems import (
    box_partition,
    diffusion_csr,
    gen_aniso3d,
    gen_poisson2d,
    gen_poisson3d,
    gen_skyscraper,
    make_config,
)

__version__ = "0.1.0"

__all__ = [
    "Breakdown",
    "SparseSpdMatrix",
    "spmv",
    "spmm",
    "gram",
    "cholesky_small",
    "trsm_right_inv",
    "norm2",
    "Partition",
    "contiguous_partition",
    "read_partition",
    "write_partition",
    "a_orthogonalize_against",
    "a_cholqr",
    "pre_cholqr",
    "CsrOperator",
    "as_operator",
    "StencilOperator",
    "METHODS",
    "RETENTIONS",
    "SolverConfig",
    "ConvergenceReport",
    "BasisStore",
    "enlarged_solve",
    "cg",
    "diffusion_csr",
    "gen_poisson2d",
    "gen_poisson3d",
    "gen_aniso3d",
    "gen_skyscraper",
    "box_partition",
    "make_config",
    "make_rhs",
    "run_batch",
    "run_experiment",
    "write_history",
    "write_runs_csv",
    "CSV_COLUMNS",
    "BlockJacobiFactor",
    "uniform_block_bounds",
    "build_block_jacobi",
    "forward_solve",
    "backward_solve",
    "apply_minv",
    "aligned_with",
]
