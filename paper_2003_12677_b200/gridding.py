"""Host views of the gridding matrix in the reference's own vocabulary
(gridding.py:33-195): SparseCOO, prune, coo_to_csr, build_coo, build_matrix.

The matrices themselves are assembled on the device (sptb_build.cu) and live
in the plan; these functions copy them out for callers that inspect or export
them.  ``build_coo`` returns the entries the device kept -- the reference's
raw triplets without its out-of-grid sentinel rows and with threshold-0
zeros already dropped -- so ``prune`` is a no-op on it and
``coo_to_csr(prune(build_coo(...)))`` equals the reference's build_matrix.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cache import HostGridCSR as SparseGridCSR
from .cache import build_matrix

SENTINEL_ROW = -1


@dataclass
class SparseCOO:
    """Triplet form (gridding.py:33-45); rows may hold the sentinel -1."""

    shape: tuple
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.size)


def build_coo(geom, spec, sample_weights=None) -> SparseCOO:
    """Triplets of S (rows = F-order grid index, cols = samples), from the device build."""
    m = build_matrix(geom, spec, sample_weights)
    rows = np.repeat(np.arange(m.shape[0], dtype=np.int64), np.diff(m.row_ptr))
    return SparseCOO(shape=m.shape, rows=rows, cols=m.col_idx.copy(), vals=m.vals.copy())


def prune(coo: SparseCOO, threshold: float = 0.0) -> SparseCOO:
    """Drop sentinel rows and |val| <= threshold (gridding.py:159-163)."""
    keep = (coo.rows != SENTINEL_ROW) & (np.abs(coo.vals) > threshold)
    return SparseCOO(shape=coo.shape, rows=coo.rows[keep], cols=coo.cols[keep], vals=coo.vals[keep])


def coo_to_csr(coo: SparseCOO) -> SparseGridCSR:
    """Canonical CSR plus the materialised conjugate transpose (gridding.py:166-188)."""
    import scipy.sparse as sp
    if np.any(coo.rows == SENTINEL_ROW):
        raise ValueError("COO still contains sentinel rows; call prune() first")
    m = sp.coo_matrix((coo.vals.astype(np.complex128), (coo.rows, coo.cols)), shape=coo.shape).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    madj = m.conj().transpose().tocsr()
    madj.sum_duplicates()
    madj.sort_indices()
    return SparseGridCSR(coo.shape, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data,
                         madj.indptr.astype(np.int64), madj.indices.astype(np.int64), madj.data)
