"""B200-native ASDSM (Anisotropic Submeshes Domain Splitting Method) solver.

The product is ``libasdsm_b200.so`` (CUDA kernels for sm_100a behind the C-ABI in
``include/asdsm_b200.h``).  This package is a thin ctypes mirror of the reference's C++
solver/driver interface (proj/include/asdsm/*.hpp) so callers and tests read like the
reference's own.  There is no CPU fallback: without the built library or a GPU every
solve raises.
"""
from .asdsm import (  # noqa: F401
    DegenerateError,
    DimensionMismatch,
    DivisibilityError,
    Error,
    IndexOutOfRange,
    InvalidKind,
    IterateOptions,
    IterationRecord,
    IterationState,
    MeshConfig,
    MeshKind,
    NoExactSolution,
    NotASubmesh,
    Problem,
    ProblemSpec,
    SingularMatrix,
    SkeletonNotHollow,
    SolverContext,
    UnknownExample,
    Unsupported,
    ZeroNormSolution,
    RunConfig,
    RunResult,
    asdsm_iterate,
    example_mesh,
    format_history_csv,
    residual_snapshot,
    run_experiment,
    write_text_file,
    baseline_mesh,
    baseline_problem,
    build_projector,
    hole_positions,
    library_path,
    load_library,
    make_problem,
)
