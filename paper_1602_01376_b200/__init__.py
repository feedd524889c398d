"""B200-native Inv-ASKIT factorization and solve (arXiv 1602.01376).

Drop-in for the reference's hot path (`kernelsolve.factorize`, `solve`,
`solve_many`; /root/reference/pkg/src/kernelsolve/solver.py:92-237): the
operator's inputs (tree, skeletons, interpolation matrices) come from the
reference compression, and the factor/solve runs in libinvaskit.so
(hand-written sm_100a CUDA, C ABI in include/invaskit.h).
"""

from .errors import (
    DataFormatError,
    DeviceError,
    IllConditionedError,
    InvalidArgumentError,
    KernelSolveError,
    NotSPDError,
    SingularMatrixError,
)
from .problem import Problem, as_problem, from_arrays, from_compressed_kernel
from .krr import krr_fit, krr_predict
from .persist import load_factor, load_operator, load_points, save_factor, save_operator, save_points
from .solver import GpuHierFactor, factorize, hss_matvec, release_cached_memory, solve, solve_many

HierFactor = GpuHierFactor

__all__ = [
    "DataFormatError",
    "DeviceError",
    "GpuHierFactor",
    "HierFactor",
    "IllConditionedError",
    "InvalidArgumentError",
    "KernelSolveError",
    "NotSPDError",
    "Problem",
    "SingularMatrixError",
    "as_problem",
    "factorize",
    "release_cached_memory",
    "from_arrays",
    "from_compressed_kernel",
    "hss_matvec",
    "krr_fit",
    "krr_predict",
    "load_factor",
    "load_operator",
    "load_points",
    "save_factor",
    "save_operator",
    "save_points",
    "solve",
    "solve_many",
]
