"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/sptb.h declares, and the host-side API mirrors the reference's
validation and planning semantics (no device compute here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sptb.h")).read()
    return sorted(set(re.findall(r"\b(sptb_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    import paper_2003_12677_b200 as sb
    lib = ctypes.CDLL(sb.LIB_PATH)
    missing = [s for s in _declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(_declared_symbols()) >= 20


def test_library_is_sm100a():
    import subprocess
    import paper_2003_12677_b200 as sb
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ctypes_signatures_cover_header():
    from paper_2003_12677_b200 import _lib
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(_declared_symbols()) <= bound


def test_version_and_error_string():
    from paper_2003_12677_b200 import _lib
    assert _lib.lib.sptb_version() >= 1
    assert isinstance(_lib.last_error(), str)


def test_plan_create_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any device call."""
    from paper_2003_12677_b200 import _lib
    h = ctypes.c_void_p()
    ct = np.ones(4)
    st = np.zeros(4)
    g = _lib.Geometry(1, 4, 16, 16, 0.5, ct.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                      st.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    k = _lib.Kernel(0, 3, 5.0, 0.5)
    rc = _lib.lib.sptb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 0, 32, 0, 0.0)
    assert rc == _lib.ERR_ARG
    g.n_p = 16
    k.width = 4
    assert _lib.lib.sptb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 0, 32, 0, 0.0) == _lib.ERR_ARG
    k.width = 3
    assert _lib.lib.sptb_plan_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(k), 0, 12, 0, 0.0) == _lib.ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(_lib.ERR_ARG, "x")


@pytest.mark.parametrize("kwargs", [
    dict(n_p=1, n_theta=4), dict(n_p=8, n_theta=0), dict(n_p=8, n_theta=4, n_z=0),
    dict(n_p=8, n_theta=4, center=8.0), dict(n_p=8, n_theta=4, center=-0.1),
    dict(n_p=8, n_theta=4, angles=np.zeros(3)), dict(n_p=8, n_theta=2, angles=np.array([0.0, 7.0])),
])
def test_scan_geometry_validation(kwargs):
    """test_geometry.py:27-38."""
    from paper_2003_12677_b200 import ScanGeometry
    with pytest.raises(ValueError):
        ScanGeometry(**kwargs)


def test_scan_geometry_defaults():
    from paper_2003_12677_b200 import ScanGeometry
    g = ScanGeometry(n_p=16, n_theta=12)
    assert g.n_x == g.n_y == 16 and g.center == 8.0
    assert g.grid_shape == (16, 16) and g.sino_shape == (12, 16)
    assert list(ScanGeometry(n_p=8, n_theta=1).signed_freqs()) == [0, 1, 2, 3, -4, -3, -2, -1]


@pytest.mark.parametrize("bad", [dict(family="spline"), dict(width=2), dict(width=-1),
                                 dict(beta=0.0), dict(family="gauss", sigma=-1.0)])
def test_kernel_spec_validation(bad):
    from paper_2003_12677_b200 import KernelSpec
    with pytest.raises(ValueError):
        KernelSpec(**bad)


def test_filters_match_oracle():
    from oracle import OGeom, filter_weights
    from paper_2003_12677_b200 import ScanGeometry, make_filter, sample_weights
    for n in (16, 17, 32):
        g = ScanGeometry(n_p=n, n_theta=3)
        for kind in ("none", "ramlak", "shepplogan", "hamming"):
            np.testing.assert_array_equal(make_filter(kind, g).weights,
                                          filter_weights(kind, OGeom(n, 3)))
    g = ScanGeometry(n_p=8, n_theta=3)
    w = sample_weights(make_filter("ramlak", g), g)
    assert w.shape == (24,)
    with pytest.raises(ValueError):
        make_filter("density", g)


@pytest.mark.parametrize("kwargs", [{"algorithm": "emission"}, {"max_iter": 0}, {"tol": -1e-3},
                                    {"mu": 0.0}, {"mu": -2.0}, {"tv_inner_iter": 0}])
def test_solver_config_validation(kwargs):
    from paper_2003_12677_b200 import SolverConfig
    with pytest.raises(ValueError):
        SolverConfig(**kwargs)


def test_solver_config_filter_defaults():
    from paper_2003_12677_b200 import SolverConfig
    assert SolverConfig(algorithm="fbp").filter_kind() == "ramlak"
    assert SolverConfig(algorithm="sirt").filter_kind() == "hamming"
    assert SolverConfig(algorithm="cgls").filter_kind() == "none"
    assert SolverConfig(algorithm="tv").filter_kind() == "none"


def test_plan_chunks_semantics():
    """test_pipeline.py:30-74."""
    from paper_2003_12677_b200 import plan_chunks
    assert plan_chunks(10, 4).passes[0] == ((0, 3), (3, 3), (6, 2), (8, 2))
    p = plan_chunks(20, 4, max_per_pass=2)
    assert [[r[1] for r in row] for row in p.passes] == [[2, 2, 2, 2], [2, 2, 2, 2], [1, 1, 1, 1]]
    assert [r[1] for r in plan_chunks(3, 4).nonempty_ranges()] == [1, 1, 1]
    rng = np.random.default_rng(11)
    for _ in range(30):
        n_z, w, per = int(rng.integers(1, 60)), int(rng.integers(1, 7)), int(rng.integers(1, 9))
        cursor = 0
        for row in plan_chunks(n_z, w, per).passes:
            lens = [ln for _, ln in row]
            assert max(lens) - min(lens) <= 1 and lens == sorted(lens, reverse=True)
            for start, ln in row:
                assert ln <= per and start == cursor
                cursor += ln
        assert cursor == n_z
    for bad in ({"n_z": 0, "workers": 1}, {"n_z": 4, "workers": 0},
                {"n_z": 4, "workers": 1, "max_per_pass": 0}):
        with pytest.raises(ValueError):
            plan_chunks(**bad)


def test_pairing_roundtrip():
    from paper_2003_12677_b200 import ShapeMismatchError, pair_complex, unpair
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((2, 5, 7))
    ra, rb = unpair(pair_complex(a, b))
    np.testing.assert_array_equal(ra, a)
    np.testing.assert_array_equal(rb, b)
    with pytest.raises(ShapeMismatchError):
        pair_complex(np.ones((2, 3)), np.ones((3, 2)))


def test_stack_validation():
    from paper_2003_12677_b200 import (ScanGeometry, ShapeMismatchError, SinogramStack,
                                       TomogramStack)
    geom = ScanGeometry(n_p=16, n_theta=5, n_z=2)
    with pytest.raises(ShapeMismatchError):
        SinogramStack(data=np.zeros((2, 5, 17)), geometry=geom)
    with pytest.raises(ShapeMismatchError):
        SinogramStack(data=np.zeros((5, 16)), geometry=geom)
    with pytest.raises(ShapeMismatchError):
        TomogramStack(data=np.zeros((4, 4)))


def test_errors_mirror_reference_hierarchy():
    import paper_2003_12677_b200 as sb
    for name in ("ShapeMismatchError", "NearZeroDenominatorError", "DivergenceError",
                 "NonFiniteError", "WorkerFailureError", "CorruptCacheError"):
        assert issubclass(getattr(sb, name), sb.SptomoError)
    e = sb.WorkerFailureError((0, 4), "NonFiniteError('x')")
    assert e.slice_range == (0, 4) and "NonFinite" in str(e.cause)
