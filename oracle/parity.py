"""Parallel oracle evaluation for parity checks at production sizes -- TEST
INFRASTRUCTURE ONLY (used by tests/ and bench.py's parity self-check, never
by the product path).

At 2048^2 x 1536 one oracle operator application costs ~1 s and one solver
iteration ~2 s per complex pair on one core, so the parity checks at the
headline configuration evaluate their few pairs concurrently: a fork pool
whose workers inherit the already-built oracle operators (the reference's
pipeline does the same, pipeline.py:163,206).
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from .solvers import o_solve

_STATE: dict = {}


def _job(args):
    kind, key, payload, kw = args
    ops = _STATE[key]
    if kind == "iradon":
        return ops.iradon(payload)
    if kind == "radon":
        return ops.radon(payload)
    if kind == "radon_adjoint":
        return ops.radon_adjoint(payload)
    if kind == "solve":
        algo = kw.pop("algorithm")
        u, rep = o_solve(payload, ops, algo, **kw)
        return u, list(rep.history), rep.iterations, rep.converged
    raise ValueError(kind)


def register(key: str, ops) -> None:
    """Make ``ops`` visible to pool workers forked after this call."""
    _STATE[key] = ops


def run(jobs, processes: int | None = None):
    """Evaluate ``jobs`` = [(kind, key, input, kwargs)] in a fork pool of at
    most one process per job; results in job order."""
    if not jobs:
        return []
    n = min(len(jobs), processes or os.cpu_count() or 1)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if n == 1:
        return [_job(j) for j in jobs]
    with mp.get_context("fork").Pool(processes=n) as pool:
        return pool.map(_job, jobs, chunksize=1)


def pair_of(x: np.ndarray, k: int) -> np.ndarray:
    """Complex pair unit k of a real stack: x[2k] + i x[2k+1] (pipeline.py:36-47)."""
    return x[2 * k].astype(np.float64) + 1j * x[2 * k + 1].astype(np.float64)


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    b = np.asarray(b, dtype=np.complex128 if np.iscomplexobj(b) else np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
