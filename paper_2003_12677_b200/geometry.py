"""Scan geometry and kernel specification (API of sptomo/geometry.py).

Only the parameter objects live here; the numerics that consume them (polar
sample positions, kernel weights, deapodization) run inside libsptb when a
plan is built (csrc/sptb_build.cu restates geometry.py:146-272).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _frozen_f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class ScanGeometry:
    """Parallel-beam layout (geometry.py:32-111): n_p detector bins, n_theta
    angles in [0, 2 pi) (default: evenly over [0, pi)), n_z slices, an
    n_y x n_x grid (default n_p x n_p) and the rotation-axis column
    ``center`` (default n_p / 2)."""

    n_p: int
    n_theta: int
    angles: np.ndarray = None
    n_z: int = 1
    n_x: int = None
    n_y: int = None
    center: float = None

    def __post_init__(self):
        set_ = object.__setattr__
        for name, low in (("n_p", 2), ("n_theta", 1), ("n_z", 1)):
            if getattr(self, name) < low:
                raise ValueError(f"{name} must be >= {low}, got {getattr(self, name)}")
        ang = (np.linspace(0.0, np.pi, self.n_theta, endpoint=False)
               if self.angles is None else np.atleast_1d(self.angles))
        ang = _frozen_f64(ang)
        if ang.shape != (self.n_theta,):
            raise ValueError(f"angles has shape {ang.shape}, expected ({self.n_theta},)")
        if ang.size and (ang.min() < 0.0 or ang.max() >= 2.0 * np.pi):
            raise ValueError("angles must lie in [0, 2*pi)")
        set_(self, "angles", ang)
        set_(self, "n_x", self.n_p if self.n_x is None else int(self.n_x))
        set_(self, "n_y", self.n_p if self.n_y is None else int(self.n_y))
        if min(self.n_x, self.n_y) < 2:
            raise ValueError("n_x and n_y must be >= 2")
        set_(self, "center", self.n_p / 2.0 if self.center is None else float(self.center))
        if not 0.0 <= self.center < self.n_p:
            raise ValueError(f"center must satisfy 0 <= center < n_p, got {self.center}")

    @property
    def grid_shape(self) -> tuple:
        return (self.n_y, self.n_x)

    @property
    def sino_shape(self) -> tuple:
        return (self.n_theta, self.n_p)

    @property
    def n_samples(self) -> int:
        return self.n_theta * self.n_p

    @property
    def n_grid(self) -> int:
        return self.n_x * self.n_y

    def signed_freqs(self) -> np.ndarray:
        """FFT-order signed detector frequencies."""
        half = self.n_p // 2
        return ((np.arange(self.n_p) + half) % self.n_p - half).astype(np.float64)


@dataclass(frozen=True)
class KernelSpec:
    """Separable gridding kernel (geometry.py:115-143): Kaiser-Bessel
    (beta default 2.5 (width-1)) or truncated Gaussian (sigma default
    width/6); width odd."""

    family: str = "kb"
    width: int = 3
    beta: float = None
    sigma: float = None

    def __post_init__(self):
        if self.family not in ("kb", "gauss"):
            raise ValueError(f"unknown kernel family {self.family!r}")
        if self.width < 1 or self.width % 2 == 0:
            raise ValueError(f"kernel width must be odd and >= 1, got {self.width}")
        if self.beta is None:
            object.__setattr__(self, "beta", 2.5 * (self.width - 1))
        if self.sigma is None:
            object.__setattr__(self, "sigma", self.width / 6.0)
        if self.beta <= 0 or self.sigma <= 0:
            raise ValueError("beta and sigma must be positive")

    def cache_token(self) -> str:
        return f"{self.family}:{self.width}:{self.beta!r}:{self.sigma!r}"


@dataclass(frozen=True)
class Deapodization:
    """Real-space kernel correction (geometry.py:218-235); values are the
    plan's host copy, both arrays read-only."""

    values: np.ndarray
    support_mask: np.ndarray

    def __post_init__(self):
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        m = np.ascontiguousarray(self.support_mask, dtype=bool)
        v.setflags(write=False)
        m.setflags(write=False)
        object.__setattr__(self, "values", v)
        object.__setattr__(self, "support_mask", m)


def support_mask(geom) -> np.ndarray:
    """Inscribed disk, radius min(n_x, n_y)/2, strict (geometry.py:238-244)."""
    dy = np.arange(geom.n_y)[:, None] - geom.n_y / 2.0
    dx = np.arange(geom.n_x)[None, :] - geom.n_x / 2.0
    r = min(geom.n_x, geom.n_y) / 2.0
    return dy * dy + dx * dx < r * r


def checkerboard(geom) -> np.ndarray:
    """(-1)^(x+y) with +1 at (n_y//2, n_x//2) (geometry.py:247-251)."""
    ix = np.arange(geom.n_x)[None, :] - geom.n_x // 2
    iy = np.arange(geom.n_y)[:, None] - geom.n_y // 2
    return 1.0 - 2.0 * ((ix + iy) % 2)


# ------------------------------------------------------------------ reference helpers
# Setup-time math the reference exposes (geometry.py:146-272).  Nothing on the
# device path calls these: the plan evaluates the kernel, its transform and the
# deapodization in sptb_build.cu; they are here so callers of the reference
# API find the same functions.


def kernel_eval(spec: KernelSpec, t) -> np.ndarray:
    """K(t), exact zero for |t| >= width/2, K(0) = 1 (geometry.py:146-161)."""
    from scipy.special import i0
    t = np.asarray(t, dtype=np.float64)
    inside = np.abs(t) < spec.width / 2.0
    ts = np.where(inside, t, 0.0)
    if spec.family == "kb":
        arg = 1.0 - (2.0 * ts / spec.width) ** 2
        vals = i0(spec.beta * np.sqrt(np.maximum(arg, 0.0))) / i0(spec.beta)
    else:
        vals = np.exp(-0.5 * (ts / spec.sigma) ** 2)
    return np.where(inside, vals, 0.0)


def kernel_transform(spec: KernelSpec, nu) -> np.ndarray:
    """Continuous Fourier transform of the kernel (geometry.py:164-191): KB in
    closed form (sinh / sin branch), Gaussian by 64-point Gauss-Legendre."""
    from scipy.special import i0
    nu = np.asarray(nu, dtype=np.float64)
    if spec.family == "kb":
        w = float(spec.width)
        z2 = spec.beta ** 2 - (np.pi * w * nu) ** 2
        pos = z2 > 0
        zp = np.sqrt(np.where(pos, z2, 1.0))
        zn = np.sqrt(np.where(pos, 1.0, -z2))
        small = np.abs(zn) < 1e-12
        sn = np.where(small, 1.0, np.sin(np.where(small, 1.0, zn)) / np.where(small, 1.0, zn))
        return np.where(pos, np.sinh(zp) / zp, sn) * (w / i0(spec.beta))
    half = spec.width / 2.0
    nodes, weights = np.polynomial.legendre.leggauss(64)
    t = nodes * half
    k = np.exp(-0.5 * (t / spec.sigma) ** 2) * weights * half
    return np.cos(2.0 * np.pi * np.multiply.outer(nu, t)) @ k


def stencil_offsets(width: int):
    """(s_x, s_y) over the width^2 stencil, s_x slowest (geometry.py:194-199)."""
    h = width // 2
    r = np.arange(-h, h + 1)
    sx, sy = np.meshgrid(r, r, indexing="ij")
    return sx.ravel(), sy.ravel()


def polar_coords(geom) -> np.ndarray:
    """(N, 2) Fourier-plane positions p (cos t, sin t) + (n_x/2, n_y/2),
    theta-major (geometry.py:202-215)."""
    p = geom.signed_freqs()
    px = np.multiply.outer(np.cos(geom.angles), p) + geom.n_x / 2.0
    py = np.multiply.outer(np.sin(geom.angles), p) + geom.n_y / 2.0
    return np.stack([px.ravel(), py.ravel()], axis=1)


def deapodization_compute(geom, spec: KernelSpec) -> Deapodization:
    """The plan's deapodization (geometry.py:254-272), computed by the device
    build (NearZeroDenominatorError like the reference)."""
    from .operators import _deapo_only
    return _deapo_only(geom, spec)
