"""Drop-in operator layer (API of sptomo/operators.py) over libsptb.

``build_operators`` builds a device plan (gridding matrices, deapodization,
folded filter, calibration) and returns a ``TomoOperators`` whose members
have the reference's names, shapes and real/complex semantics
(operators.py:240-299).  Arrays may be NumPy (host, float64/complex128 in
and out, like the reference) or CUDA torch tensors (device-resident, output
dtype follows the input); leading batch dimensions are accepted as an
extension.  All arithmetic runs in libsptb on the GPU -- there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from . import cache as _cachemod
from .errors import CorruptCacheError, ShapeMismatchError
from .geometry import Deapodization, KernelSpec, ScanGeometry, support_mask

FILTER_KINDS = ("none", "ramlak", "shepplogan", "hamming", "density")
PRECISIONS = {"complex64": _lib.PREC_F32, "complex128": _lib.PREC_F64}

try:  # torch is optional plumbing: device tensors + the current CUDA stream
    import torch
except Exception:  # pragma: no cover - torch is in the image
    torch = None


# ------------------------------------------------------------------ filters


@dataclass
class FilterSpec:
    """Fourier weights for backprojection / preconditioning
    (operators.py:28-49): radial (n_p) or per-sample (n_theta*n_p)."""

    kind: str
    weights: np.ndarray
    residual_history: np.ndarray = None
    converged: bool = True
    final_residual: float = None

    def __post_init__(self):
        if self.kind not in FILTER_KINDS:
            raise ValueError(f"unknown filter kind {self.kind!r}")
        w = np.asarray(self.weights, dtype=np.float64)
        if np.any(w < 0) or not np.all(np.isfinite(w)):
            raise ValueError("filter weights must be finite and >= 0")
        self.weights = w


def make_filter(kind: str, geom) -> FilterSpec:
    """ramlak |f|, shepplogan |f| sinc f, hamming |f|(0.54 + 0.46 cos 2 pi f),
    none 1, over f = signed_freq / n_p in FFT order (operators.py:52-71)."""
    if kind == "density":
        raise ValueError("density weights are produced by density_filter_solve")
    half = geom.n_p // 2
    f = ((np.arange(geom.n_p) + half) % geom.n_p - half) / geom.n_p
    shapes = {
        "none": lambda: np.ones(geom.n_p),
        "ramlak": lambda: np.abs(f),
        "shepplogan": lambda: np.abs(f) * np.sinc(f),
        "hamming": lambda: np.abs(f) * (0.54 + 0.46 * np.cos(2.0 * np.pi * f)),
    }
    if kind not in shapes:
        raise ValueError(f"unknown filter kind {kind!r}")
    return FilterSpec(kind=kind, weights=shapes[kind]())


def sample_weights(filt: FilterSpec, geom) -> np.ndarray:
    """Per-sample weights, radial filters tiled over angles (operators.py:74-82)."""
    w = filt.weights
    if w.shape == (geom.n_samples,):
        return w
    if w.shape == (geom.n_p,):
        return np.tile(w, geom.n_theta)
    raise ShapeMismatchError(f"filter weights shape {w.shape} fits neither (n_p,) nor (N,)")


@dataclass(frozen=True)
class Preconditioner:
    """Diagonal detector-axis weights (operators.py:85-96)."""

    weights: np.ndarray

    def __post_init__(self):
        w = np.ascontiguousarray(self.weights, dtype=np.float64)
        if np.any(w < 0) or not np.all(np.isfinite(w)):
            raise ValueError("preconditioner weights must be finite and >= 0")
        w.setflags(write=False)
        object.__setattr__(self, "weights", w)


def density_filter_solve(csr, geom, max_iter: int = 50, tol: float = 1e-6) -> FilterSpec:
    """Least-squares sample weights that flatten the gridded response
    (operators.py:189-236): CGLS on || |S| d - 1 ||_2, clamped >= 0 and
    symmetrised in p, computed on the device from the plan's CSR pair."""
    plan = csr._plan
    if plan.precision != _lib.PREC_F64:
        # the least-squares problem is ill-conditioned (50 CGLS steps amplify
        # complex64 rounding of |S| ~1e5x): solve on a complex128 build of the
        # same matrices, like the reference, and fold the weights into ours
        plan = _Plan(plan.geom, plan.kernel, _lib.PREC_F64, 1, plan.device, plan.threshold)
    n = geom.n_theta * geom.n_p
    w = np.empty(n, dtype=np.float64)
    hist = np.empty(int(max_iter) + 1, dtype=np.float64)
    nh, conv, fin = C.c_int32(), C.c_int32(), C.c_double()
    check(lib.sptb_density_filter(plan.h, int(max_iter), float(tol),
                                  w.ctypes.data_as(C.POINTER(C.c_double)),
                                  hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nh),
                                  C.byref(conv), C.byref(fin)), "density_filter_solve")
    return FilterSpec(kind="density", weights=w, residual_history=hist[:nh.value].copy(),
                      converged=bool(conv.value), final_residual=float(fin.value))


# ------------------------------------------------------------------ device plan


class _Plan:
    """Owns one libsptb plan (matrices + deapodization + work buffers)."""

    def __init__(self, geom, kernel, precision, max_batch, device, threshold):
        ct = np.ascontiguousarray(np.cos(geom.angles), dtype=np.float64)
        st = np.ascontiguousarray(np.sin(geom.angles), dtype=np.float64)
        g = _lib.Geometry(geom.n_p, geom.n_theta, geom.n_x, geom.n_y, float(geom.center),
                          ct.ctypes.data_as(C.POINTER(C.c_double)),
                          st.ctypes.data_as(C.POINTER(C.c_double)))
        fam = {"kb": _lib.KERNEL_KB, "gauss": _lib.KERNEL_GAUSS}[kernel.family]
        k = _lib.Kernel(fam, int(kernel.width), float(kernel.beta), float(kernel.sigma))
        h = C.c_void_p()
        check(lib.sptb_plan_create(C.byref(h), C.byref(g), C.byref(k), precision, max_batch,
                                   device, float(threshold)), "build_operators")
        self.h = h
        self.geom = geom
        self.kernel = kernel
        self.threshold = threshold
        self.precision = precision
        self.device = device
        self.max_batch = max_batch
        self.filter_w = None   # per-sample or radial weights folded into S diag(w), or None
        self.calib = 1.0       # the plan's iradon calibration (reset by set_filter)

    def set_filter(self, w):
        if w is None:
            check(lib.sptb_plan_set_filter(self.h, None, 0))
            self.filter_w = None
            self.calib = 1.0
            return
        w = np.ascontiguousarray(w, dtype=np.float64).ravel()
        check(lib.sptb_plan_set_filter(self.h, w.ctypes.data_as(C.POINTER(C.c_double)), w.size),
              "set_filter")
        self.filter_w = w
        self.calib = 1.0

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib.sptb_plan_destroy(h)
            self.h = None

    def matrix_info(self, which):
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.sptb_plan_matrix_info(self.h, which, C.byref(r), C.byref(c), C.byref(n)))
        return r.value, c.value, n.value

    def bind_stream(self, stream_ptr):
        check(lib.sptb_plan_set_stream(self.h, C.c_void_p(stream_ptr)))


def _is_cuda_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _apply(plan: _Plan, fn, x, in_shape, out_shape, what, extra=()):
    """Run one C-ABI operator on numpy (host) or CUDA-tensor (device) input."""
    if _is_cuda_tensor(x):
        if tuple(x.shape[-2:]) != tuple(in_shape):
            raise ShapeMismatchError(f"{what} shape {tuple(x.shape)} != {in_shape}")
        t = x.contiguous()
        cplx = t.is_complex()
        if t.dtype in (torch.float32, torch.complex64):
            fmt = _lib.FMT_F32
        elif t.dtype in (torch.float64, torch.complex128):
            fmt = _lib.FMT_F64
        else:
            t = t.to(torch.float32)
            fmt = _lib.FMT_F32
        fmt |= _lib.FMT_COMPLEX if cplx else _lib.FMT_REAL
        lead = tuple(t.shape[:-2])
        n = int(np.prod(lead)) if lead else 1
        out = torch.empty(lead + tuple(out_shape), dtype=t.dtype, device=t.device)
        if n:
            plan.bind_stream(torch.cuda.current_stream(t.device).cuda_stream)
            check(fn(plan.h, *extra, C.c_void_p(t.data_ptr()), fmt, C.c_void_p(out.data_ptr()),
                     fmt, n), what)
        return out
    a = np.asarray(x.cpu().numpy() if torch is not None and isinstance(x, torch.Tensor) else x)
    if a.shape[-2:] != tuple(in_shape) or a.ndim < 2:
        raise ShapeMismatchError(f"{what} shape {a.shape} != {tuple(in_shape)}")
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    fmt = _lib.FMT_F64 | (_lib.FMT_COMPLEX if cplx else _lib.FMT_REAL)
    lead = a.shape[:-2]
    n = int(np.prod(lead)) if lead else 1
    out = np.empty(lead + tuple(out_shape), dtype=a.dtype)
    if n:
        plan.bind_stream(0)
        check(fn(plan.h, *extra, a.ctypes.data_as(C.c_void_p), fmt,
                 out.ctypes.data_as(C.c_void_p), fmt, n), what)
    return out


# ------------------------------------------------------------------ matrices


class DeviceGridCSR:
    """Handle on a plan-resident gridding matrix (stands in for
    SparseGridCSR, gridding.py:47-81).  ``shape``/``nnz`` are cheap; the host
    CSR arrays in the reference's index convention are materialised lazily
    for inspection (``row_ptr``, ``col_idx``, ``vals``, ``adj_*``,
    ``matrix``, ``adjoint``)."""

    def __init__(self, plan: _Plan, filtered: bool):
        self._plan = plan
        self.filtered = filtered
        rows, cols, nnz = plan.matrix_info(_lib.MAT_S)
        self.shape = (rows, cols)
        self._nnz = nnz
        self._host = None

    @property
    def nnz(self) -> int:
        # the filtered matrix shares S's pattern on the device; its reference
        # counterpart drops the entries the folded weights zero (or push to
        # <= threshold), so its nnz comes from the pruned host view
        if self.filtered:
            return int(self.matrix.nnz)
        return self._nnz

    def _fetch(self):
        if self._host is not None:
            return self._host
        import scipy.sparse as sp
        g = self._plan.geom
        rows, cols = self.shape
        rp = np.empty(rows + 1, dtype=np.int32)
        ci = np.empty(max(self._nnz, 1), dtype=np.int32)
        v = np.empty(2 * max(self._nnz, 1), dtype=np.float64)
        which = _lib.MAT_SW if self.filtered else _lib.MAT_S
        check(lib.sptb_plan_matrix_copy(self._plan.h, which, rp.ctypes.data_as(C.c_void_p),
                                        ci.ctypes.data_as(C.c_void_p),
                                        v.ctypes.data_as(C.c_void_p)))
        vals = (v[0::2] + 1j * v[1::2])[: self._nnz]
        # device rows are row-major grid points m = y*n_x + x; the reference
        # uses x*n_y + y (gridding.py:10-11)
        mc = np.arange(rows)
        mf = (mc % g.n_x) * g.n_y + mc // g.n_x
        lens = np.diff(rp)
        coo_r = np.repeat(mf, lens)
        S = sp.csr_matrix((vals, (coo_r, ci[: self._nnz])), shape=self.shape)
        S.sum_duplicates()
        if self.filtered:  # the reference's folded build prunes |w v| <= threshold (gridding.py:159-163)
            thr = self._plan.threshold
            if thr > 0:
                S.data[np.abs(S.data) <= thr] = 0.0
            S.eliminate_zeros()
        S.sort_indices()
        SH = S.conj().T.tocsr()
        SH.sort_indices()
        self._host = (S, SH)
        return self._host

    @property
    def matrix(self):
        return self._fetch()[0]

    @property
    def adjoint(self):
        return self._fetch()[1]

    row_ptr = property(lambda s: s.matrix.indptr.astype(np.int64))
    col_idx = property(lambda s: s.matrix.indices.astype(np.int64))
    vals = property(lambda s: s.matrix.data)
    adj_row_ptr = property(lambda s: s.adjoint.indptr.astype(np.int64))
    adj_col_idx = property(lambda s: s.adjoint.indices.astype(np.int64))
    adj_vals = property(lambda s: s.adjoint.data)


def spmv(csr: DeviceGridCSR, x, adjoint: bool = False):
    """y = S x or S^H x on the device (operators.py:124-129)."""
    rows, cols = csr.shape
    want = rows if adjoint else cols
    a = np.asarray(x)
    if a.shape[0] != want:
        raise ShapeMismatchError(f"x has {a.shape[0]} rows, matrix wants {want}")
    vec = a.ndim == 1
    a2 = np.ascontiguousarray(a.reshape(want, -1), dtype=np.complex128)
    out_rows = cols if adjoint else rows
    y = np.empty((out_rows, a2.shape[1]), dtype=np.complex128)
    which = _lib.MAT_SH if adjoint else (_lib.MAT_SW if csr.filtered else _lib.MAT_S)
    csr._plan.bind_stream(0)
    check(lib.sptb_spmm(csr._plan.h, which, a2.ctypes.data_as(C.c_void_p),
                        y.ctypes.data_as(C.c_void_p), a2.shape[1],
                        _lib.FMT_F64 | _lib.FMT_COMPLEX), "spmv")
    return y[:, 0] if vec else y


def spmm(csr: DeviceGridCSR, x, adjoint: bool = False):
    """Multi-column spmv; x is (cols, n_rhs) (operators.py:132-136)."""
    if np.ndim(x) != 2:
        raise ShapeMismatchError("spmm expects a 2D right-hand side")
    return spmv(csr, x, adjoint=adjoint)


# ------------------------------------------------------------------ free functions


def radon(tomo, csr: DeviceGridCSR, deapo=None, geom=None):
    """Forward projection (operators.py:153-168) through csr's plan."""
    p = csr._plan
    return _apply(p, lib.sptb_radon, tomo, p.geom.grid_shape, p.geom.sino_shape, "tomogram")


def iradon(sino, csr: DeviceGridCSR, deapo=None, geom=None, weights=None, scale: float = 1.0):
    """Backprojection (operators.py:171-187): csr_filtered carries the folded
    filter; explicit ``weights`` ((n_p,) or (N,)) are folded into the plan for
    this call when they differ from its current filter, then restored."""
    p = csr._plan
    if weights is None:
        return _apply(p, lib.sptb_backproject, sino, p.geom.sino_shape, p.geom.grid_shape,
                      "sinogram", extra=(1 if csr.filtered else 0, C.c_double(scale)))
    w = np.ascontiguousarray(weights, dtype=np.float64).ravel()
    if w.size not in (p.geom.n_p, p.geom.n_theta * p.geom.n_p):
        raise ShapeMismatchError(f"weights of size {w.size} fit neither (n_p,) nor (N,)")
    keep, keep_calib = p.filter_w, p.calib
    same = keep is not None and keep.size == w.size and np.array_equal(keep, w)
    if not same:
        p.set_filter(w)
    try:
        return _apply(p, lib.sptb_backproject, sino, p.geom.sino_shape, p.geom.grid_shape,
                      "sinogram", extra=(1, C.c_double(scale)))
    finally:
        if not same:
            p.set_filter(keep)
            check(lib.sptb_plan_set_calibration(p.h, C.c_double(keep_calib)))
            p.calib = keep_calib


def _spectral(plan, sino, w):
    w = np.ascontiguousarray(w, dtype=np.float64).ravel()
    return _apply(plan, lib.sptb_spectral_apply, sino, plan.geom.sino_shape,
                  plan.geom.sino_shape, "sinogram",
                  extra=(w.ctypes.data_as(C.POINTER(C.c_double)), w.size))


# ------------------------------------------------------------------ bundle


@dataclass
class TomoOperators:
    """Matched operator bundle (operators.py:239-299), plan-backed."""

    geom: ScanGeometry
    kernel: KernelSpec
    deapo: Deapodization
    csr: DeviceGridCSR
    filter_spec: FilterSpec | None
    csr_filtered: DeviceGridCSR | None
    filter_weights: np.ndarray | None
    calib_scale: float = 1.0
    _plan: _Plan = None

    @property
    def plan(self) -> _Plan:
        return self._plan

    def radon(self, tomo):
        return _apply(self._plan, lib.sptb_radon, tomo, self.geom.grid_shape,
                      self.geom.sino_shape, "tomogram")

    def radon_adjoint(self, sino):
        return _apply(self._plan, lib.sptb_radon_adjoint, sino, self.geom.sino_shape,
                      self.geom.grid_shape, "sinogram")

    def iradon(self, sino):
        if self.filter_spec is None or self.filter_spec.kind == "none":
            return self.radon_adjoint(sino)
        return _apply(self._plan, lib.sptb_iradon, sino, self.geom.sino_shape,
                      self.geom.grid_shape, "sinogram")

    def preconditioner(self, kind: str = "hamming") -> Preconditioner:
        if kind == "none":
            return Preconditioner(weights=np.ones(self.geom.n_p))
        return Preconditioner(weights=make_filter(kind, self.geom).weights)

    @property
    def spectral_weights(self) -> np.ndarray:
        if self.filter_spec is None or self.filter_spec.kind == "none":
            return np.ones(self.geom.n_p)
        w = self.filter_spec.weights
        if w.shape == (self.geom.n_p,):
            return w
        return w.reshape(self.geom.sino_shape)

    def precondition(self, sino):
        return precondition_apply(Preconditioner(weights=self.spectral_weights), sino, self)

    def apply_weights(self, sino):
        return _spectral(self._plan, sino, self.spectral_weights)


_SPECTRAL_PLANS: dict = {}


def _spectral_plan(n_theta: int, n_p: int, like) -> _Plan:
    """A device plan for detector-axis spectral passes over (n_theta, n_p)
    sinograms, cached per (shape, precision, device): precondition_apply has
    no operator bundle in the reference's signature."""
    prec = _lib.PREC_F64
    if _is_cuda_tensor(like) and like.dtype in (torch.float32, torch.complex64):
        prec = _lib.PREC_F32
    dev = like.device.index if _is_cuda_tensor(like) else _default_device()
    key = (int(n_theta), int(n_p), prec, dev)
    plan = _SPECTRAL_PLANS.get(key)
    if plan is None:
        plan = _Plan(ScanGeometry(n_p=int(n_p), n_theta=int(n_theta)), KernelSpec(), prec, 8, dev, 0.0)
        _SPECTRAL_PLANS[key] = plan
    return plan


def precondition_apply(pre: Preconditioner, sino, ops: TomoOperators | None = None):
    """Half-power preconditioner: detector-axis spectrum times sqrt(weights)
    (operators.py:108-121).  Same signature as the reference; the FFT pair
    runs on the device through ``ops``' plan when given (and of matching
    shape), else through a cached plan for the sinogram's shape.  Weights
    may be radial (n_p,) or per sample, shaped like the sinogram."""
    sh = tuple(np.shape(sino))
    if len(sh) == 0 or sh[-1] != pre.weights.shape[-1]:
        raise ShapeMismatchError(f"sinogram last axis {sh[-1] if sh else None} != weights "
                                 f"{pre.weights.shape[-1]}")
    w = np.sqrt(pre.weights)
    x = sino
    if len(sh) == 1:  # one detector row
        x = sino[None]
    shape2 = tuple(np.shape(x))[-2:]
    if w.ndim > 1 and tuple(w.shape) != shape2:
        raise ShapeMismatchError(f"weights shape {w.shape} != sinogram {shape2}")
    plan = ops._plan if ops is not None and tuple(ops.geom.sino_shape) == shape2 else None
    if plan is None:
        plan = _spectral_plan(shape2[0], shape2[1], x)
    wc = np.ascontiguousarray(w, dtype=np.float64).ravel()
    out = _apply(plan, lib.sptb_spectral_apply, x, shape2, shape2, "sinogram",
                 extra=(wc.ctypes.data_as(C.POINTER(C.c_double)), int(wc.size)))
    return out[0] if len(sh) == 1 else out


def _default_device():
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0


def _deapo_only(geom, kernel):
    plan = _Plan(geom, kernel, _lib.PREC_F64, 1, _default_device(), 0.0)
    dv = np.empty(geom.grid_shape, dtype=np.float64)
    check(lib.sptb_plan_deapo_copy(plan.h, dv.ctypes.data_as(C.c_void_p)))
    return Deapodization(values=dv, support_mask=support_mask(geom))


def _cache_matrix(plan, dev_csr, geom, kernel, filter_id, weights, cache_dir):
    """SGCSR001 cache entry for this matrix (operators.py:329-337): validate an
    existing file (CorruptCacheError like the reference) and check it describes
    the same matrix as the device build; store one when missing, with
    complex128 values from a complex128 build."""
    key = _cachemod.make_cache_key(geom, kernel, filter_id)
    found = _cachemod.cache_check(key, cache_dir)
    prune = weights is not None
    if found is None:
        src = dev_csr
        if plan.precision != _lib.PREC_F64:
            p64 = _Plan(geom, kernel, _lib.PREC_F64, 1, plan.device, plan.threshold)
            if weights is not None:
                p64.set_filter(weights)
            src = DeviceGridCSR(p64, filtered=weights is not None)
        _cachemod.cache_store(key, _cachemod.host_csr(src, prune), cache_dir)
    else:
        rows, cols, nnz = found
        if (rows, cols) != tuple(dev_csr.shape):
            raise CorruptCacheError(f"{_cachemod.cache_path(key, cache_dir)}: shape "
                                    f"{(rows, cols)} disagrees with the geometry")
    return key


def build_operators(geom, kernel: KernelSpec | None = None, filter_kind: str = "ramlak",
                    cache_dir: str | None = None, fold_filter: bool = True,
                    threshold: float = 0.0, *, precision: str = "complex64",
                    max_batch: int = 32, device: int | None = None) -> TomoOperators:
    """Build the device plan (operators.py:317-371).  The matrices are
    assembled on the GPU in well under a second; ``cache_dir`` keeps the
    reference's SGCSR001 files and calibration meta compatible both ways
    (cache.py); ``fold_filter`` only changes what the bundle reports (the
    device always folds)."""
    if kernel is None:
        kernel = KernelSpec()
    if filter_kind not in FILTER_KINDS:
        raise ValueError(f"unknown filter kind {filter_kind!r}")
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    plan = _Plan(geom, kernel, PRECISIONS[precision], int(max_batch),
                 _default_device() if device is None else int(device), threshold)
    dv = np.empty(geom.grid_shape, dtype=np.float64)
    check(lib.sptb_plan_deapo_copy(plan.h, dv.ctypes.data_as(C.c_void_p)))
    deapo = Deapodization(values=dv, support_mask=support_mask(geom))
    csr = DeviceGridCSR(plan, filtered=False)
    if cache_dir is not None:
        _cache_matrix(plan, csr, geom, kernel, "none", None, cache_dir)
    filter_spec = None
    csr_f = None
    weights = None
    calib = 1.0
    if filter_kind != "none":
        if filter_kind == "density":
            filter_spec = density_filter_solve(csr, geom)
        else:
            filter_spec = make_filter(filter_kind, geom)
        weights = sample_weights(filter_spec, geom)
        plan.set_filter(filter_spec.weights)
        csr_f = DeviceGridCSR(plan, filtered=True)
        cached = None
        if cache_dir is not None and fold_filter:
            key_f = _cache_matrix(plan, csr_f, geom, kernel, filter_kind, filter_spec.weights, cache_dir)
            cached = _cachemod.read_calib(key_f, cache_dir)
        if cached is not None:  # operators.py:355-359
            calib = cached
            check(lib.sptb_plan_set_calibration(plan.h, C.c_double(calib)))
        else:
            c = C.c_double()
            check(lib.sptb_plan_calibrate(plan.h, C.byref(c)), "calibration")
            calib = c.value
            if cache_dir is not None and fold_filter:
                _cachemod.write_calib(key_f, cache_dir, calib)
        plan.calib = calib
    else:
        plan.set_filter(None)
    return TomoOperators(geom=geom, kernel=kernel, deapo=deapo, csr=csr,
                         filter_spec=filter_spec, csr_filtered=csr_f if fold_filter else None,
                         filter_weights=None if fold_filter else weights,
                         calib_scale=calib, _plan=plan)
