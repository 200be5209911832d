"""B200-native sketched Hessenberg (sCMRH) / sketched LSLU (sLSLU) iteration
loop of arXiv 2502.02721, behind the reference package's own entry points.

    from paper_2502_02721_b200 import LinearOperator, SolverConfig, slslu
    res = slslu(LinearOperator.from_matrix(A), b, SolverConfig(maxiter=30))

The loop runs as hand-written sm_100a CUDA kernels behind the C ABI in
``include/hessketch_b200.h`` (library built in-tree by ``build.py``).  There is
no CPU fallback: without the library or a GPU every solve raises.
"""

from .hessenberg import (
    DeviceFactorization,
    GeneralizedHessenbergState,
    HessenbergState,
    PivotStrategy,
    TrivialSolution,
    dump_factorization,
    init_generalized,
    init_square,
    pivot_select,
    step_generalized,
    step_square,
)
from .linops import (
    CsrOperator,
    DenseOperator,
    DeviceOperator,
    LinearOperator,
    OpCounters,
    PsfOperator,
    RANK_TOL,
    RankDeficiencyError,
    TomographyOperator,
    dense_qr_ls,
    stacked_tikhonov_ls,
    to_device_operator,
)
from .sketch import (
    DeviceSketch,
    GaussianSketch,
    SketchOperator,
    SparseSignSketch,
    derive_seed,
    device_sketch,
    make_gaussian_sketch,
    sketch_apply,
)
from .solvers import (
    CSV_COLUMNS,
    SOLVERS,
    SolveResult,
    SolverConfig,
    SolverTrace,
    TraceRecord,
    cmrh,
    gmres,
    lslu,
    lsqr,
    pivot_positions,
    scmrh,
    scmrh_tikhonov,
    slslu,
    slslu_tikhonov,
    trace_to_csv,
)

__version__ = "0.1.0"
