"""paper_2003_12677_b200: B200-native sparse-matrix tomography operators.

Drop-in for the hot path of the reference package ``sptomo`` (arXiv
2003.12677): the gridding Radon pair, gridrec/FBP and the SIRT / CGLS / TV
solvers, computed by hand-written sm_100a CUDA kernels in ``libsptb.so``
behind a C ABI (include/sptb.h).  Importing this package loads that library;
there is no CPU fallback.
"""

from .errors import (CorruptCacheError, DivergenceError, FileFormatError,
                     GridTooLargeError, InvalidFlatFieldError,
                     NearZeroDenominatorError, NonFiniteError,
                     ShapeMismatchError, SptomoError, WorkerFailureError)
from .geometry import (Deapodization, KernelSpec, ScanGeometry, checkerboard,
                       deapodization_compute, kernel_eval, kernel_transform, polar_coords,
                       stencil_offsets, support_mask)
from .gridding import SparseCOO, build_coo, coo_to_csr, prune
from .operators import (FILTER_KINDS, DeviceGridCSR, FilterSpec, Preconditioner,
                        TomoOperators, build_operators, density_filter_solve, iradon,
                        make_filter,
                        precondition_apply, radon, sample_weights, spmm, spmv)
from .solvers import (ALGORITHMS, DEFAULT_FILTERS, SolverConfig, SolverReport,
                      solve, solve_cgls, solve_fbp, solve_sirt, solve_tv)
from .pipeline import (PAIRING_TOL, ChunkPlan, SinogramStack, TomogramStack,
                       pair_complex, plan_chunks, run_pipeline, unpair)
from ._lib import LIB_PATH, launch_count
from .cache import (CACHE_MAGIC, CACHE_VERSION, MatrixCacheKey, SparseGridCSR, build_matrix,
                    cache_load, cache_store, make_cache_key)
from .io import (KIND_INTENSITY, KIND_SINOGRAM, KIND_TOMOGRAM, VolumeFile, VolumeHeader,
                 VolumeWriter, read_header, read_volume, write_volume)

__version__ = "0.1.0"

__all__ = [
    "ALGORITHMS", "CACHE_MAGIC", "CACHE_VERSION", "ChunkPlan", "MatrixCacheKey", "cache_load",
    "cache_store", "make_cache_key", "SparseGridCSR", "build_matrix", "KIND_INTENSITY",
    "KIND_SINOGRAM", "KIND_TOMOGRAM", "VolumeFile", "VolumeHeader", "VolumeWriter",
    "read_header", "read_volume", "write_volume", "deapodization_compute", "kernel_eval", "kernel_transform",
    "polar_coords", "stencil_offsets", "SparseCOO", "build_coo", "coo_to_csr", "prune", "CorruptCacheError", "DEFAULT_FILTERS",
    "Deapodization", "density_filter_solve", "DeviceGridCSR", "DivergenceError", "FILTER_KINDS",
    "FileFormatError", "FilterSpec", "GridTooLargeError", "InvalidFlatFieldError",
    "KernelSpec", "LIB_PATH", "NearZeroDenominatorError", "NonFiniteError",
    "PAIRING_TOL", "Preconditioner", "ScanGeometry", "ShapeMismatchError",
    "SinogramStack", "SolverConfig", "SolverReport", "SptomoError",
    "TomoOperators", "TomogramStack", "WorkerFailureError", "build_operators",
    "checkerboard", "iradon", "launch_count", "make_filter", "pair_complex",
    "plan_chunks", "precondition_apply", "radon", "run_pipeline",
    "sample_weights", "solve", "solve_cgls", "solve_fbp", "solve_sirt",
    "solve_tv", "spmm", "spmv", "support_mask", "unpair",
]
