"""SGCSR001 matrix cache, file-compatible with the reference (gridding.py:196-293)
plus the calibration meta file of build_operators (operators.py:345-367).

The device builds the gridding matrices in well under a second, so the cache
is not needed for speed; it is kept for interoperability: a cache directory
written by either implementation is readable by the other, keys are the same
SHA-256 digests, and corrupt files raise ``CorruptCacheError`` exactly where
the reference does.  Files written here hold complex128 values computed by a
complex128 device build (the reference's precision), with the zero entries
that a folded zero-weight filter column produces pruned as the reference's
threshold-0 build prunes them (gridding.py:159-172).
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import tempfile
from dataclasses import dataclass

import numpy as np

from .errors import CorruptCacheError

CACHE_MAGIC = b"SGCSR001"
CACHE_VERSION = 1
_HEAD = struct.Struct("<I3Q")


@dataclass(frozen=True)
class MatrixCacheKey:
    """Content digest of everything the matrix values depend on (gridding.py:196-205)."""

    digest: str  # 64 hex chars (sha256)

    @property
    def raw(self) -> bytes:
        return bytes.fromhex(self.digest)


def make_cache_key(geom, spec, filter_id: str = "none", version: int = CACHE_VERSION) -> MatrixCacheKey:
    """gridding.py:209-217: sha256 over (version, n_p, n_theta, n_x, n_y,
    center), the angles as little-endian float64, the kernel token and the
    filter id."""
    h = hashlib.sha256()
    h.update(struct.pack("<5qd", version, geom.n_p, geom.n_theta, geom.n_x, geom.n_y, geom.center))
    h.update(np.ascontiguousarray(geom.angles, dtype="<f8").tobytes())
    h.update(spec.cache_token().encode())
    h.update(b"|" + filter_id.encode())
    return MatrixCacheKey(digest=h.hexdigest())


def cache_path(key: MatrixCacheKey, cache_dir: str) -> str:
    return os.path.join(cache_dir, key.digest + ".sgcsr")


def meta_path(key: MatrixCacheKey, cache_dir: str) -> str:
    return os.path.join(cache_dir, key.digest + ".meta.json")


@dataclass
class HostGridCSR:
    """Host copy of a cached matrix in the reference's index convention."""

    shape: tuple
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    adj_row_ptr: np.ndarray
    adj_col_idx: np.ndarray
    adj_vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.size)


def _write_block(fh, row_ptr, col_idx, vals):
    fh.write(np.ascontiguousarray(row_ptr, dtype="<u8").tobytes())
    fh.write(np.ascontiguousarray(col_idx, dtype="<u8").tobytes())
    iv = np.empty((vals.size, 2), dtype="<f8")
    iv[:, 0] = vals.real
    iv[:, 1] = vals.imag
    fh.write(iv.tobytes())


def cache_store(key: MatrixCacheKey, matrix, cache_dir: str) -> str:
    """Atomically write S and S^H under the digest name (gridding.py:232-253).
    ``matrix``: a DeviceGridCSR, a HostGridCSR or anything with the
    reference's SparseGridCSR fields."""
    os.makedirs(cache_dir, exist_ok=True)
    path = cache_path(key, cache_dir)
    rows, cols = matrix.shape
    header = CACHE_MAGIC + _HEAD.pack(CACHE_VERSION, rows, cols, matrix.nnz)
    fd, tmp = tempfile.mkstemp(dir=cache_dir, suffix=".tmp")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(header)
            fh.write(key.raw)
            _write_block(fh, matrix.row_ptr, matrix.col_idx, matrix.vals)
            _write_block(fh, matrix.adj_row_ptr, matrix.adj_col_idx, matrix.adj_vals)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return path


def _read_exact(fh, n: int, path: str) -> bytes:
    buf = fh.read(n)
    if len(buf) != n:
        raise CorruptCacheError(f"{path}: truncated (wanted {n} bytes)")
    return buf


def _header(fh, key: MatrixCacheKey, path: str):
    head = _read_exact(fh, len(CACHE_MAGIC) + _HEAD.size, path)
    if head[:8] != CACHE_MAGIC:
        raise CorruptCacheError(f"{path}: bad magic {head[:8]!r}")
    version, rows, cols, nnz = _HEAD.unpack(head[8:])
    if version != CACHE_VERSION:
        raise CorruptCacheError(f"{path}: unsupported version {version}")
    if _read_exact(fh, 32, path) != key.raw:
        raise CorruptCacheError(f"{path}: digest mismatch")
    return rows, cols, nnz


def _expected_size(rows: int, cols: int, nnz: int) -> int:
    return len(CACHE_MAGIC) + _HEAD.size + 32 + 8 * (rows + 1) + 8 * (cols + 1) + 2 * 24 * nnz


def cache_check(key: MatrixCacheKey, cache_dir: str):
    """Validate a cached file without reading its arrays: None on miss, else
    (rows, cols, nnz); CorruptCacheError on bad magic / version / digest /
    truncation / trailing bytes (the reference's checks, gridding.py:270-288)."""
    path = cache_path(key, cache_dir)
    if not os.path.exists(path):
        return None
    with open(path, "rb") as fh:
        rows, cols, nnz = _header(fh, key, path)
    size = os.path.getsize(path)
    want = _expected_size(rows, cols, nnz)
    if size < want:
        raise CorruptCacheError(f"{path}: truncated (wanted {want} bytes)")
    if size > want:
        raise CorruptCacheError(f"{path}: trailing bytes")
    return rows, cols, nnz


def cache_load(key: MatrixCacheKey, cache_dir: str) -> HostGridCSR | None:
    """Load a cached matrix (gridding.py:268-293): None on miss,
    CorruptCacheError on bad content."""
    path = cache_path(key, cache_dir)
    if not os.path.exists(path):
        return None

    def block(fh, n_rows, nnz):
        rp = np.frombuffer(_read_exact(fh, 8 * (n_rows + 1), path), dtype="<u8").astype(np.int64)
        ci = np.frombuffer(_read_exact(fh, 8 * nnz, path), dtype="<u8").astype(np.int64)
        iv = np.frombuffer(_read_exact(fh, 16 * nnz, path), dtype="<f8").reshape(nnz, 2)
        return rp, ci, iv[:, 0] + 1j * iv[:, 1]

    with open(path, "rb") as fh:
        rows, cols, nnz = _header(fh, key, path)
        rp, ci, v = block(fh, rows, nnz)
        arp, aci, av = block(fh, cols, nnz)
        if fh.read(1):
            raise CorruptCacheError(f"{path}: trailing bytes")
    if rp[-1] != nnz or arp[-1] != nnz:
        raise CorruptCacheError(f"{path}: row_ptr/nnz disagree")
    return HostGridCSR((int(rows), int(cols)), rp, ci, v, arp, aci, av)


def host_csr(dev_csr, prune_zeros: bool) -> HostGridCSR:
    """Host copy of a plan matrix in the reference's convention; explicit
    zeros dropped when the reference's threshold-0 build would not keep them."""
    S = dev_csr.matrix.tocsr()
    if prune_zeros:
        S.eliminate_zeros()
    S.sort_indices()
    SH = S.conj().T.tocsr()
    SH.sort_indices()
    return HostGridCSR(S.shape, S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data,
                       SH.indptr.astype(np.int64), SH.indices.astype(np.int64), SH.data)


SparseGridCSR = HostGridCSR  # the reference's name for the host matrix pair (gridding.py:47-81)


def build_matrix(geom, spec, weights=None, threshold: float = 0.0) -> HostGridCSR:
    """gridding.py:191-195 on the device: S and S^H (optionally S diag(w),
    zero entries pruned) assembled by a complex128 plan and copied to the host
    in the reference's index convention."""
    from . import _lib
    from .operators import DeviceGridCSR, _Plan, _default_device
    plan = _Plan(geom, spec, _lib.PREC_F64, 1, _default_device(), threshold)
    if weights is not None:
        plan.set_filter(np.asarray(weights, dtype=np.float64))
    return host_csr(DeviceGridCSR(plan, filtered=weights is not None), prune_zeros=weights is not None)


def read_calib(key: MatrixCacheKey, cache_dir: str):
    p = meta_path(key, cache_dir)
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return float(json.load(fh)["calib_scale"])


def write_calib(key: MatrixCacheKey, cache_dir: str, calib: float) -> None:
    """Atomic tmp + rename like operators.py:360-367."""
    os.makedirs(cache_dir, exist_ok=True)
    p = meta_path(key, cache_dir)
    tmp = p + f".tmp{os.getpid()}"
    with open(tmp, "w") as fh:
        json.dump({"calib_scale": calib}, fh)
    os.replace(tmp, p)
