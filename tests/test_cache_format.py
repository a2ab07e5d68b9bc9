"""SGCSR001 cache compatibility with the reference (gridding.py:196-293).

CPU: cache keys equal the reference's digests (fixtures from the unmodified
reference), store/load round trip and the corruption checks.  GPU:
build_operators(cache_dir=...) writes files whose matrices equal the
reference's CSR, reuses the calibration meta, and rejects corrupt files."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def _geom_kernel(sb, case):
    return sb.ScanGeometry(**case["geom"]), sb.KernelSpec(**case["kernel"])


def test_cache_keys_match_reference():
    import paper_2003_12677_b200.cache as cache
    from paper_2003_12677_b200.geometry import KernelSpec, ScanGeometry
    cases = json.load(open(os.path.join(GOLDEN, "cache_keys.json")))
    assert len(cases) == 36
    for c in cases:
        g, k = ScanGeometry(**c["geom"]), KernelSpec(**c["kernel"])
        assert cache.make_cache_key(g, k, c["filter"]).digest == c["digest"], c


def _host_matrix(seed=0):
    from paper_2003_12677_b200.cache import HostGridCSR
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    S = sp.random(12, 9, density=0.3, random_state=rng, format="csr") * (1 + 1j)
    S.sort_indices()
    SH = S.conj().T.tocsr()
    SH.sort_indices()
    return HostGridCSR(S.shape, S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data,
                       SH.indptr.astype(np.int64), SH.indices.astype(np.int64), SH.data)


def test_store_load_round_trip_and_corruption(tmp_path):
    import paper_2003_12677_b200.cache as cache
    from paper_2003_12677_b200.errors import CorruptCacheError
    from paper_2003_12677_b200.geometry import KernelSpec, ScanGeometry
    key = cache.make_cache_key(ScanGeometry(n_p=32, n_theta=16), KernelSpec(), "none")
    m = _host_matrix()
    path = cache.cache_store(key, m, str(tmp_path))
    back = cache.cache_load(key, str(tmp_path))
    for f in ("row_ptr", "col_idx", "vals", "adj_row_ptr", "adj_col_idx", "adj_vals"):
        np.testing.assert_array_equal(getattr(back, f), getattr(m, f))
    assert cache.cache_check(key, str(tmp_path)) == (12, 9, m.nnz)
    other = cache.make_cache_key(ScanGeometry(n_p=32, n_theta=17), KernelSpec(), "none")
    assert cache.cache_load(other, str(tmp_path)) is None
    raw = open(path, "rb").read()
    for bad in (b"XXXXXXXX" + raw[8:], raw[:-5], raw + b"\0"):
        open(path, "wb").write(bad)
        with pytest.raises(CorruptCacheError):
            cache.cache_load(key, str(tmp_path))
        with pytest.raises(CorruptCacheError):
            cache.cache_check(key, str(tmp_path))


@pytest.mark.gpu
def test_build_operators_cache_is_reference_format(tmp_path):
    import paper_2003_12677_b200 as sb
    import paper_2003_12677_b200.cache as cache
    d = load_golden("ops_g32.npz")
    g = sb.ScanGeometry(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]))
    k = sb.KernelSpec()
    ops1 = sb.build_operators(g, k, filter_kind="ramlak", cache_dir=str(tmp_path))
    m = cache.cache_load(cache.make_cache_key(g, k, "none"), str(tmp_path))
    np.testing.assert_array_equal(m.row_ptr, d["S_row_ptr"])
    np.testing.assert_array_equal(m.col_idx, d["S_col_idx"])
    np.testing.assert_allclose(m.vals, d["S_vals"], rtol=0, atol=1e-14)
    np.testing.assert_array_equal(m.adj_row_ptr, d["SH_row_ptr"])
    mf = cache.cache_load(cache.make_cache_key(g, k, "ramlak"), str(tmp_path))
    assert mf.nnz == m.nnz - g.n_theta * 9   # the zero-weight DC column is pruned
    key_f = cache.make_cache_key(g, k, "ramlak")
    assert cache.read_calib(key_f, str(tmp_path)) == pytest.approx(ops1.calib_scale, rel=1e-12)
    # second build: calibration from the meta file
    cache.write_calib(key_f, str(tmp_path), 0.5)
    ops2 = sb.build_operators(g, k, filter_kind="ramlak", cache_dir=str(tmp_path))
    assert ops2.calib_scale == 0.5
    p = cache.cache_path(cache.make_cache_key(g, k, "none"), str(tmp_path))
    open(p, "r+b").write(b"BADMAGIC")
    with pytest.raises(sb.CorruptCacheError):
        sb.build_operators(g, k, filter_kind="none", cache_dir=str(tmp_path))


@pytest.mark.gpu
def test_gridding_host_views_match_reference():
    import paper_2003_12677_b200 as sb
    d = load_golden("ops_g32.npz")
    g = sb.ScanGeometry(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]))
    k = sb.KernelSpec()
    m = sb.coo_to_csr(sb.prune(sb.build_coo(g, k)))
    np.testing.assert_array_equal(m.row_ptr, d["S_row_ptr"])
    np.testing.assert_array_equal(m.col_idx, d["S_col_idx"])
    np.testing.assert_allclose(m.vals, d["S_vals"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(sb.deapodization_compute(g, k).values, d["deapo"], rtol=1e-12)
