"""Single-precision emulations of the oracle operators (TEST INFRASTRUCTURE ONLY).

The reference algorithm is fp64 throughout; a complex64 device path cannot
track it more closely than the algorithm's own sensitivity to single-
precision operators.  Two emulations measure that floor:

* ``Fp32Operators`` rounds every operator input and output to fp32 but
  computes the operator in fp64 (an optimistic floor: a perfectly rounded
  fp32 operator);
* ``Fp32PipelineOperators`` runs the whole operator pipeline (deapodization,
  FFTs, sparse products) in complex64 like a real fp32 implementation.

Solver vector arithmetic stays fp64 in both (as on the device for CGLS/TV).
SURVEY section 7 (hard part 6) and BASELINE.md section 5 discuss the result.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .tomo import _gamma


def _r(x):
    if np.iscomplexobj(x):
        return x.astype(np.complex64).astype(np.complex128)
    return x.astype(np.float32).astype(np.float64)


class Fp32Operators:
    def __init__(self, ops):
        self.o = ops
        self.g = ops.g

    def radon(self, u):
        return _r(self.o.radon(_r(u)))

    def radon_adjoint(self, s):
        return _r(self.o.radon_adjoint(_r(s)))

    def iradon(self, s):
        return _r(self.o.iradon(_r(s)))

    def apply_weights(self, s):
        return _r(self.o.apply_weights(_r(s)))

    @property
    def spectral_weights(self):
        return self.o.w


class Fp32PipelineOperators:
    """operators.py:153-187,293-299 evaluated in complex64 end to end."""

    def __init__(self, ops):
        self.o = ops
        self.g = ops.g
        self.SH = ops.grid.SH.astype(np.complex64)
        self.S = ops.grid.S.astype(np.complex64)
        self.Sf = ops.grid_f.S.astype(np.complex64) if ops.grid_f is not None else None
        self.d = ops.deapo.astype(np.float32)
        self.gm = np.float32(_gamma(ops.g))
        self.w = np.asarray(ops.w, dtype=np.float32)

    def radon(self, u):
        cplx = np.iscomplexobj(u)
        spec = np.fft.fft2((self.d * u).astype(np.complex64), norm="ortho")
        q = self.SH @ spec.reshape(-1, order="F")
        s = np.fft.ifft(q.reshape(self.g.sino), axis=1, norm="ortho") * self.gm
        s = s.astype(np.complex128)
        return s if cplx else s.real

    def _back(self, s, S, scale):
        cplx = np.iscomplexobj(s)
        q = np.fft.fft(np.asarray(s).astype(np.complex64), axis=1, norm="ortho").reshape(-1)
        v = (S @ q).reshape(self.g.grid, order="F")
        rec = (self.d * np.fft.ifft2(v, norm="ortho") * np.float32(self.gm * scale)).astype(np.complex128)
        return rec if cplx else rec.real

    def radon_adjoint(self, s):
        return self._back(s, self.S, 1.0)

    def iradon(self, s):
        if self.Sf is None:
            return self.radon_adjoint(s)
        return self._back(s, self.Sf, self.o.calib)

    def apply_weights(self, s):
        cplx = np.iscomplexobj(s)
        f = np.fft.fft(np.asarray(s).astype(np.complex64), axis=-1, norm="ortho") * self.w
        out = np.fft.ifft(f, axis=-1, norm="ortho").astype(np.complex128)
        return out if cplx else out.real

    @property
    def spectral_weights(self):
        return self.o.w


__all__ = ["Fp32Operators", "Fp32PipelineOperators", "sp"]


class PerturbedOperators:
    """Exact fp64 operators whose outputs carry a seeded additive
    perturbation of relative (normwise) size ``eps``: a stand-in for another
    implementation whose operators agree with the reference to ``eps``.  It
    measures how far that alone moves an ill-conditioned recurrence (CGS on
    the unfiltered normal equations moves by ~1e-5 at eps = 1e-15 and ~1e-3
    at eps = 1e-13 in 8 iterations)."""

    def __init__(self, ops, eps: float, seed: int):
        self.o = ops
        self.g = ops.g
        self.eps = eps
        self.rng = np.random.default_rng(seed)

    def _p(self, x):
        x = np.asarray(x)
        n = self.rng.standard_normal(x.shape)
        if np.iscomplexobj(x):
            n = n + 1j * self.rng.standard_normal(x.shape)
        return x + (self.eps * np.linalg.norm(x) / np.sqrt(max(x.size, 1))) * n

    def radon(self, u):
        return self._p(self.o.radon(u))

    def radon_adjoint(self, s):
        return self._p(self.o.radon_adjoint(s))

    def iradon(self, s):
        return self._p(self.o.iradon(s))

    def apply_weights(self, s):
        return self.o.apply_weights(s)

    @property
    def spectral_weights(self):
        return self.o.w
