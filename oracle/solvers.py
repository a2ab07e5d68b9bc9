"""Oracle restatement of the reconstruction solvers (TEST INFRASTRUCTURE ONLY).

Per-channel semantics follow reference solvers.py: a complex input carries
two real slices (real / imaginary channel) and every scalar is computed per
channel (solvers.py:1-10, 71-119).  The oracle keeps the reference's
complex128 representation so its iterates match the reference's bit for bit
in structure and to fp64 rounding in value.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DIVERGENCE = 10.0  # solvers.py:27


class ODivergence(RuntimeError):
    """Residual above 10x its running minimum (solvers.py:169-172)."""


class ONonFinite(RuntimeError):
    """NaN/Inf in an iterate (solvers.py:111-113, 445-447)."""


@dataclass
class OReport:
    history: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False


def _chans(a):
    return (a.real, a.imag) if np.iscomplexobj(a) else (a,)


def cdot(a, b) -> np.ndarray:
    """Per-channel real inner products (solvers.py:71-80)."""
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        a = np.asarray(a, dtype=complex)
        b = np.asarray(b, dtype=complex)
    return np.array([float(np.dot(np.ravel(x), np.ravel(y)))
                     for x, y in zip(_chans(a), _chans(b))])


def cscale(al: np.ndarray, v):
    """Scale channel c by al[c] (solvers.py:83-87)."""
    if al.size == 2:
        return al[0] * v.real + 1j * (al[1] * v.imag)
    return al[0] * v


def wnorms(r, w) -> np.ndarray:
    """sqrt(sum w |F_ortho ch|^2) per channel, FFT along the last axis
    (solvers.py:90-97)."""
    return np.array([float(np.sqrt(np.sum(w * np.abs(np.fft.fft(c, axis=-1, norm="ortho")) ** 2)))
                     for c in _chans(r)])


def rss(v) -> float:
    return float(np.sqrt(np.sum(np.asarray(v) ** 2)))


def sdiv(num, den, fb):
    """num/den where den > 0, fallback elsewhere (solvers.py:104-108)."""
    out = np.array(fb, dtype=float, copy=True)
    m = den > 0
    out[m] = num[m] / den[m]
    return out


def _finite(u, what):
    if not np.all(np.isfinite(u)):
        raise ONonFinite(f"{what} produced non-finite values")


def _nonneg(u):
    if np.iscomplexobj(u):
        return np.maximum(u.real, 0.0) + 1j * np.maximum(u.imag, 0.0)
    return np.maximum(u, 0.0)


def o_fbp(sino, ops):
    """iradon + weighted residual of its reprojection (solvers.py:122-130)."""
    rec = ops.iradon(sino)
    res = rss(wnorms(ops.radon(rec) - sino, ops.spectral_weights))
    _finite(rec, "fbp")
    return rec, OReport([res], 1, True)


def o_sirt(sino, ops, max_iter, tol=0.0, bb=True, nonneg=False):
    """BB-stepped preconditioned descent (solvers.py:133-186)."""
    w = ops.spectral_weights
    cplx = np.iscomplexobj(sino)
    u = np.zeros(ops.g.grid, dtype=complex if cplx else float)
    bn = wnorms(sino, w)
    rep = OReport()
    if rss(bn) == 0.0:
        rep.converged = True
        return u, rep
    grad = ops.radon_adjoint(ops.apply_weights(sino))
    a0 = sdiv(cdot(grad, grad), wnorms(ops.radon(grad), w) ** 2, np.zeros(bn.size))
    al = a0
    best = np.inf
    for _ in range(max_iter):
        step = cscale(al, grad)
        u = u + step
        if nonneg:
            u = _nonneg(u)
        r = sino - ops.radon(u)
        rc = wnorms(r, w)
        res = rss(rc)
        rep.history.append(res)
        rep.iterations += 1
        _finite(u, "sirt")
        best = min(best, res)
        if res > DIVERGENCE * best:
            raise ODivergence(f"sirt residual {res:.3e} > 10x {best:.3e}")
        if np.max(sdiv(rc, bn, np.zeros_like(rc))) <= tol:
            rep.converged = True
            break
        g2 = ops.radon_adjoint(ops.apply_weights(r))
        if bb:
            al = sdiv(cdot(step, step), cdot(step, grad - g2), a0)
            al = np.where(al > 0, al, a0)
        else:
            al = a0
        grad = g2
    return u, rep


def _cgls(fwd, adj, norms, b, u, iters, tol, rep):
    """CGLS recurrence with per-channel activity mask (solvers.py:189-227)."""
    r = b - fwd(u)
    s = adj(r)
    p = s.copy()
    gm = cdot(s, s)
    gm0 = gm.copy()
    bn = norms(b)
    eps2 = np.finfo(float).eps ** 2
    for _ in range(iters):
        q = fwd(p)
        dl = norms(q) ** 2
        act = (dl > 0) & (gm > eps2 * gm0)
        if not act.any():
            break
        al = np.where(act, sdiv(gm, dl, np.zeros_like(gm)), 0.0)
        u = u + cscale(al, p)
        r = r - cscale(al, q)
        rc = norms(r)
        rep.history.append(rss(rc))
        rep.iterations += 1
        _finite(u, "cgls")
        if np.max(sdiv(rc, bn, np.zeros_like(rc))) <= tol:
            rep.converged = True
            break
        s = adj(r)
        gn = cdot(s, s)
        be = np.where(act, sdiv(gn, gm, np.zeros_like(gm)), 0.0)
        gm = gn
        p = s + cscale(be, p)
    return u


def _cgs(sino, ops, iters, tol, rep):
    """Conjugate gradient squared on the normal equations A^H W A u = A^H W b
    (solvers.py:262-305): shadow residual fixed at c = A^H W b, per-channel
    rho / sigma, one residual b - A u per iteration for the report."""
    w = ops.spectral_weights

    def normal(v):
        return ops.radon_adjoint(ops.apply_weights(ops.radon(v)))

    c = ops.radon_adjoint(ops.apply_weights(sino))
    u = np.zeros_like(c)
    r, shadow, p, q = c.copy(), c.copy(), c.copy(), c.copy()
    rho = cdot(shadow, r)
    bn = wnorms(sino, w)
    for _ in range(iters):
        v = normal(p)
        sig = cdot(shadow, v)
        live = np.abs(sig) > 0
        if not live.any():
            break
        al = np.where(live, sdiv(rho, sig, np.zeros_like(rho)), 0.0)
        h = q - cscale(al, v)
        stp = q + h
        u = u + cscale(al, stp)
        r = r - cscale(al, normal(stp))
        rc = wnorms(sino - ops.radon(u), w)
        rep.history.append(rss(rc))
        rep.iterations += 1
        _finite(u, "cgs")
        if np.max(sdiv(rc, bn, np.zeros_like(rc))) <= tol:
            rep.converged = True
            break
        rn = cdot(shadow, r)
        if not (np.abs(rn) > 0).any():
            break
        be = sdiv(rn, rho, np.zeros_like(rn))
        rho = rn
        q = r + cscale(be, h)
        p = q + cscale(be, h + cscale(be, p))
    return u


def o_cgls(sino, ops, max_iter, tol=0.0, nonneg=False, cgs_mode=False):
    """CGLS on min ||sqrt(w) F (A u - b)|| (solvers.py:230-259); ``cgs_mode``
    runs the CGS recurrence on the normal equations instead (:247-248)."""
    w = ops.spectral_weights
    u = np.zeros(ops.g.grid, dtype=complex if np.iscomplexobj(sino) else float)
    rep = OReport()
    if rss(wnorms(sino, w)) == 0.0:
        rep.converged = True
        return u, rep
    if cgs_mode:
        u = _cgs(sino, ops, max_iter, tol, rep)
    else:
        u = _cgls(ops.radon, lambda r: ops.radon_adjoint(ops.apply_weights(r)),
                  lambda r: wnorms(r, w), sino, u, max_iter, tol, rep)
    if nonneg:
        u = _nonneg(u)
    return u, rep


def grad2(u):
    """Forward differences, last column/row zero (solvers.py:308-314)."""
    gx = np.zeros_like(u)
    gy = np.zeros_like(u)
    gx[:, :-1] = np.diff(u, axis=1)
    gy[:-1, :] = np.diff(u, axis=0)
    return gx, gy


def div2(vx, vy):
    """Negative adjoint of grad2 (solvers.py:317-327)."""
    out = np.zeros_like(vx)
    out[:, 0] += vx[:, 0]
    out[:, 1:-1] += vx[:, 1:-1] - vx[:, :-2]
    out[:, -1] += -vx[:, -2]
    out[0, :] += vy[0, :]
    out[1:-1, :] += vy[1:-1, :] - vy[:-2, :]
    out[-1, :] += -vy[-2, :]
    return out


def shrink(vx, vy, kap):
    """Isotropic soft shrink per channel (solvers.py:330-341)."""
    def one(ax, ay, k):
        m = np.sqrt(ax * ax + ay * ay)
        f = np.maximum(m - k, 0.0) / np.where(m > 0, m, 1.0)
        return ax * f, ay * f
    if np.iscomplexobj(vx):
        ax, ay = one(vx.real, vy.real, kap[0])
        bx, by = one(vx.imag, vy.imag, kap[-1])
        return ax + 1j * bx, ay + 1j * by
    return one(vx, vy, kap[0])


def o_tv(sino, ops, max_iter, inner=2, mu=None, tol=0.0, nonneg=False):
    """Split-Bregman TV with stacked CGLS inner solves (solvers.py:344-460)."""
    w = ops.spectral_weights
    cplx = np.iscomplexobj(sino)
    nch = 2 if cplx else 1
    dt = complex if cplx else float
    bn = wnorms(sino, w)
    u = np.zeros(ops.g.grid, dtype=dt)
    rep = OReport()
    if rss(bn) == 0.0:
        rep.converged = True
        return u, rep
    if mu is not None:
        mus = np.full(nch, float(mu))
    else:
        bp = ops.radon_adjoint(sino)
        mus = 0.1 * np.array([np.max(np.abs(c)) for c in _chans(bp)])
        mus = np.where(mus > 0, mus, 1.0)
    lam = 2.0 * mus
    smu, slam = np.sqrt(mus), np.sqrt(lam)
    dx = np.zeros(ops.g.grid, dtype=dt)
    dy = np.zeros_like(dx)
    bx = np.zeros_like(dx)
    by = np.zeros_like(dx)

    def fwd(v):
        gx, gy = grad2(v)
        return [cscale(smu, ops.radon(v)), cscale(slam, gx), cscale(slam, gy)]

    def adj(t):
        return (ops.radon_adjoint(ops.apply_weights(cscale(smu, t[0])))
                - div2(cscale(slam, t[1]), cscale(slam, t[2])))

    def norms(t):
        return np.sqrt(wnorms(t[0], w) ** 2 + cdot(t[1], t[1]) + cdot(t[2], t[2]))

    for _ in range(max_iter):
        tgt = [cscale(smu, sino), cscale(slam, dx - bx), cscale(slam, dy - by)]
        # stacked CGLS (solvers.py:435-460)
        f0 = fwd(u)
        r = [a - b for a, b in zip(tgt, f0)]
        s = adj(r)
        p = s.copy()
        gm = cdot(s, s)
        for _ in range(inner):
            q = fwd(p)
            dl = norms(q) ** 2
            if not (np.all(np.isfinite(dl)) and np.all(np.isfinite(gm))):
                raise ONonFinite("tv quadratic subproblem overflowed")
            act = dl > 0
            if not act.any():
                break
            al = np.where(act, sdiv(gm, dl, np.zeros_like(gm)), 0.0)
            u = u + cscale(al, p)
            r = [a - cscale(al, b) for a, b in zip(r, q)]
            s = adj(r)
            gn = cdot(s, s)
            be = np.where(act, sdiv(gn, gm, np.zeros_like(gm)), 0.0)
            gm = gn
            p = s + cscale(be, p)
        if nonneg:
            u = _nonneg(u)
        _finite(u, "tv")
        gx, gy = grad2(u)
        dx, dy = shrink(gx + bx, gy + by, 1.0 / lam)
        bx = bx + gx - dx
        by = by + gy - dy
        rc = wnorms(sino - ops.radon(u), w)
        rep.history.append(rss(rc))
        rep.iterations += 1
        if tol > 0 and np.max(sdiv(rc, bn, np.zeros_like(rc))) <= tol:
            rep.converged = True
            break
    else:
        rep.converged = True
    return u, rep


def o_solve(sino, ops, algorithm, max_iter=10, **kw):
    """Dispatch (solvers.py:463-473)."""
    if algorithm == "fbp":
        return o_fbp(sino, ops)
    if algorithm == "sirt":
        return o_sirt(sino, ops, max_iter, **kw)
    if algorithm == "cgls":
        return o_cgls(sino, ops, max_iter, **kw)
    if algorithm == "tv":
        return o_tv(sino, ops, max_iter, **kw)
    raise ValueError(algorithm)
