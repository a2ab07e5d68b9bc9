"""SPTOMO01 volume files and the io helpers against fixtures written by the
unmodified reference (io.py:35-193)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def test_read_reference_volumes():
    from paper_2003_12677_b200 import io
    v = io.read_volume(os.path.join(GOLDEN, "vol_sino.sptomo"))
    assert v.kind == io.KIND_SINOGRAM and v.data.shape == (3, 5, 8) and v.center == 3.5
    np.testing.assert_allclose(v.angles, np.linspace(0, np.pi, 5, endpoint=False), rtol=0, atol=0)
    g = io.sinogram_geometry(v)
    assert (g.n_z, g.n_theta, g.n_p, g.center) == (3, 5, 8, 3.5)
    t = io.read_volume(os.path.join(GOLDEN, "vol_tomo.sptomo"))
    assert t.kind == io.KIND_TOMOGRAM and t.angles is None and t.data.shape == (2, 8, 8)


def test_write_is_byte_identical(tmp_path):
    from paper_2003_12677_b200 import io
    for name in ("vol_sino.sptomo", "vol_tomo.sptomo"):
        v = io.read_volume(os.path.join(GOLDEN, name))
        out = str(tmp_path / name)
        io.write_volume(out, v.kind, v.data, center=v.center, angles=v.angles)
        assert open(out, "rb").read() == open(os.path.join(GOLDEN, name), "rb").read()


def test_corrupt_volumes(tmp_path):
    from paper_2003_12677_b200 import io
    from paper_2003_12677_b200.errors import FileFormatError
    raw = open(os.path.join(GOLDEN, "vol_sino.sptomo"), "rb").read()
    for bad in (b"NOTAVOL!" + raw[8:], raw[:-3], raw + b"x"):
        p = str(tmp_path / "bad.sptomo")
        open(p, "wb").write(bad)
        with pytest.raises(FileFormatError):
            io.read_volume(p)


def test_helpers_match_reference():
    from paper_2003_12677_b200 import io
    d = load_golden("io_misc.npz")
    np.testing.assert_array_equal(io.phantom_shepp_logan(16, 3), d["phantom"])
    sino = io.read_volume(os.path.join(GOLDEN, "vol_sino.sptomo")).data
    np.testing.assert_allclose(io.normalize(np.abs(sino) + 0.1, 2.0), d["norm"], rtol=1e-15)
    with pytest.raises(Exception):
        io.normalize(sino, 0.0)


def test_geometry_helpers_against_oracle():
    """kernel_eval / kernel_transform / polar_coords restate the same
    reference lines as the oracle (geometry.py:146-215)."""
    import oracle.tomo as ot
    from paper_2003_12677_b200 import geometry as gm
    for fam in ("kb", "gauss"):
        k = gm.KernelSpec(family=fam, width=5)
        ok = ot.OKernel(family=fam, width=5)
        t = np.linspace(-3, 3, 61)
        np.testing.assert_allclose(gm.kernel_eval(k, t), ot.kernel_values(ok, t), rtol=1e-14, atol=0)
        nu = np.linspace(-0.6, 0.6, 25)
        np.testing.assert_allclose(gm.kernel_transform(k, nu), ot.kernel_ft(ok, nu), rtol=1e-12)
    g = gm.ScanGeometry(n_p=16, n_theta=5)
    sx, sy = gm.stencil_offsets(3)
    assert list(sx) == [-1, -1, -1, 0, 0, 0, 1, 1, 1] and list(sy) == [-1, 0, 1] * 3
    pc = gm.polar_coords(g)
    assert pc.shape == (80, 2)
    np.testing.assert_allclose(pc[:16, 0], g.signed_freqs() + 8.0)
