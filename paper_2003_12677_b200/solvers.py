"""Reconstruction solvers (API of sptomo/solvers.py) running on the device.

FBP, SIRT (Hamming-preconditioned, Barzilai-Borwein steps), CGLS and
split-Bregman TV are executed by ``sptb_solve`` (csrc/sptb_solvers.cu):
iterates stay resident in HBM, the sinogram-space residual is kept in the
detector-frequency domain (so the 1D FFT pair of every radon/residual step
cancels), and every per-channel scalar of the reference (solvers.py:67-119)
is computed on the device for each complex pair of a batch.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import DivergenceError, NonFiniteError, ShapeMismatchError
from .operators import TomoOperators, _is_cuda_tensor, torch

ALGORITHMS = ("fbp", "sirt", "cgls", "tv")
DEFAULT_FILTERS = {"fbp": "ramlak", "sirt": "hamming", "cgls": "none", "tv": "none"}
DIVERGENCE_FACTOR = 10.0


@dataclass
class SolverConfig:
    """Solver options with the reference's validation (solvers.py:31-56)."""

    algorithm: str = "fbp"
    max_iter: int = 10
    tol: float = 0.0
    mu: float | None = None
    tv_inner_iter: int = 2
    bb_enabled: bool = True
    filter: str | None = None
    seed: int = 0
    cgs_mode: bool = False
    nonneg: bool = False

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.tol < 0:
            raise ValueError("tol must be >= 0")
        if self.mu is not None and self.mu <= 0:
            raise ValueError("mu must be > 0")
        if self.tv_inner_iter < 1:
            raise ValueError("tv_inner_iter must be >= 1")

    def filter_kind(self) -> str:
        return self.filter if self.filter is not None else DEFAULT_FILTERS[self.algorithm]


@dataclass
class SolverReport:
    residual_history: list = field(default_factory=list)
    iterations_run: int = 0
    converged: bool = False
    wall_time: float = 0.0


_EXC = {_lib.ERR_DIVERGENCE: DivergenceError, _lib.ERR_NONFINITE: NonFiniteError}


def solve_batch(sino, ops: TomoOperators, cfg: SolverConfig, raise_on_failure: bool = True,
                out=None):
    """Solve every unit of ``sino`` ((..., n_theta, n_p), real slices paired
    (2k, 2k+1) or complex pairs) in device batches.

    Returns ``(rec, reports, status)``: one SolverReport and one status code
    per unit (0 ok, or the DivergenceError / NonFiniteError code).  With
    ``raise_on_failure`` the first failing unit raises its exception type.
    ``out``: for host input, a float32 / float64 array of the result's shape
    to write into (e.g. a memory-mapped output volume) instead of a new
    float64 array.
    """
    t0 = time.perf_counter()
    g = ops.geom
    cfg_c = _lib.SolverConfig(_lib.ALGO[cfg.algorithm], int(cfg.max_iter), float(cfg.tol),
                              float(cfg.mu) if cfg.mu is not None else 0.0,
                              int(cfg.tv_inner_iter), int(bool(cfg.bb_enabled)),
                              int(bool(cfg.nonneg)), int(bool(cfg.cgs_mode)))
    plan = ops.plan
    if _is_cuda_tensor(sino):
        if tuple(sino.shape[-2:]) != g.sino_shape:
            raise ShapeMismatchError(f"sinogram shape {tuple(sino.shape)} != {g.sino_shape}")
        t = sino.contiguous()
        cplx = t.is_complex()
        if t.dtype not in (torch.float32, torch.float64, torch.complex64, torch.complex128):
            t = t.to(torch.float32)
        fmt = (_lib.FMT_F64 if t.dtype in (torch.float64, torch.complex128) else _lib.FMT_F32)
        fmt |= _lib.FMT_COMPLEX if cplx else _lib.FMT_REAL
        lead = tuple(t.shape[:-2])
        out = torch.empty(lead + g.grid_shape, dtype=t.dtype, device=t.device)
        plan.bind_stream(torch.cuda.current_stream(t.device).cuda_stream)
        src, dst = C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr())
    else:
        a = np.asarray(sino)
        if a.ndim < 2 or a.shape[-2:] != g.sino_shape:
            raise ShapeMismatchError(f"sinogram shape {a.shape} != {g.sino_shape}")
        cplx = np.iscomplexobj(a)
        # float32 host stacks go in as they are (no float64 copy); results
        # are float64 / complex128 like the reference's
        if a.dtype == (np.complex64 if cplx else np.float32):
            a = np.ascontiguousarray(a)
            fmt_in = _lib.FMT_F32
        else:
            a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
            fmt_in = _lib.FMT_F64
        kind = _lib.FMT_COMPLEX if cplx else _lib.FMT_REAL
        lead = a.shape[:-2]
        fmt_o = _lib.FMT_F64
        if out is None:
            out = np.empty(lead + g.grid_shape, dtype=np.complex128 if cplx else np.float64)
        else:
            want = (np.complex64, np.complex128) if cplx else (np.float32, np.float64)
            if out.shape != lead + g.grid_shape or out.dtype not in want or not out.flags.c_contiguous:
                raise ShapeMismatchError(f"out must be a C-contiguous {lead + g.grid_shape} array of "
                                         f"{'/'.join(str(np.dtype(d)) for d in want)}")
            fmt_o = _lib.FMT_F32 if out.dtype in (np.float32, np.complex64) else _lib.FMT_F64
        plan.bind_stream(0)
        src, dst = a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)
        t = a
        fmt = None
    n = int(np.prod(lead)) if lead else 1
    units = n if cplx else (n + 1) // 2
    iters_cap = 1 if cfg.algorithm == "fbp" else int(cfg.max_iter)
    hist = np.zeros((max(units, 1), iters_cap), dtype=np.float64)
    its = np.zeros(max(units, 1), dtype=np.int32)
    conv = np.zeros(max(units, 1), dtype=np.int32)
    stat = np.zeros(max(units, 1), dtype=np.int32)
    fmt_out = fmt if fmt is not None else fmt_o | kind
    fmt_src = fmt if fmt is not None else fmt_in | kind
    rc = lib.sptb_solve(plan.h, C.byref(cfg_c), src, fmt_src, dst, fmt_out, n,
                        hist.ctypes.data_as(C.c_void_p), its.ctypes.data_as(C.c_void_p),
                        conv.ctypes.data_as(C.c_void_p), stat.ctypes.data_as(C.c_void_p))
    if rc not in (_lib.OK, _lib.ERR_DIVERGENCE, _lib.ERR_NONFINITE):
        check(rc, f"solve_{cfg.algorithm}")
    msg = _lib.last_error()
    wall = time.perf_counter() - t0
    reports = [SolverReport(residual_history=[float(v) for v in hist[u, :its[u]]],
                            iterations_run=int(its[u]), converged=bool(conv[u]),
                            wall_time=wall) for u in range(units)]
    if raise_on_failure:
        for u in range(units):
            if stat[u] != _lib.OK:
                raise _EXC.get(int(stat[u]), RuntimeError)(
                    f"{cfg.algorithm} unit {u}: {msg}")
    return out, reports, [int(s) for s in stat[:units]]


def _single(sino, ops, cfg):
    rec, reps, _ = solve_batch(sino, ops, cfg)
    nd = sino.ndim if hasattr(sino, "ndim") else np.ndim(sino)
    if nd == 2:
        return rec, reps[0]
    return rec, reps


def solve_fbp(sino, ops: TomoOperators):
    """Calibrated iradon + weighted residual of its reprojection
    (solvers.py:122-130)."""
    return _single(sino, ops, SolverConfig(algorithm="fbp", max_iter=1))


def solve_sirt(sino, ops: TomoOperators, cfg: SolverConfig):
    """BB-stepped SIRT with divergence guard (solvers.py:133-186)."""
    return _single(sino, ops, cfg)


def solve_cgls(sino, ops: TomoOperators, cfg: SolverConfig):
    """CGLS on min ||sqrt(w) F (A u - b)|| (solvers.py:230-259)."""
    return _single(sino, ops, cfg)


def solve_tv(sino, ops: TomoOperators, cfg: SolverConfig):
    """Split-Bregman TV (solvers.py:344-432)."""
    return _single(sino, ops, cfg)


def solve(sino, ops: TomoOperators, cfg: SolverConfig):
    """Dispatch on cfg.algorithm (solvers.py:463-473)."""
    if cfg.algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {cfg.algorithm!r}")
    if cfg.algorithm == "fbp":
        return solve_fbp(sino, ops)
    return _single(sino, ops, cfg)
