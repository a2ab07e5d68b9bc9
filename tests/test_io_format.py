"""SPTOMO01 volume files against fixtures written by the unmodified
reference (io.py:35-89): byte-identical writes, validated (memory-mapped)
reads, the streamed writer and the corruption checks."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def test_read_reference_volumes():
    from paper_2003_12677_b200 import io
    v = io.read_volume(os.path.join(GOLDEN, "vol_sino.sptomo"))
    assert v.kind == io.KIND_SINOGRAM and v.data.shape == (3, 5, 8) and v.center == 3.5
    np.testing.assert_allclose(v.angles, np.linspace(0, np.pi, 5, endpoint=False), rtol=0, atol=0)
    assert isinstance(v.data, np.memmap) and v.data.dtype == np.float32
    h = io.read_header(os.path.join(GOLDEN, "vol_sino.sptomo"))
    assert h.shape == (3, 5, 8) and h.payload_offset == 8 + 45 + 8 * 5
    w = io.read_volume(os.path.join(GOLDEN, "vol_sino.sptomo"), mmap=False)
    np.testing.assert_array_equal(w.data, v.data)
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


def test_streamed_writer_matches_whole_write(tmp_path):
    """Slices written out of order (as ranks / chunks finish) give the same
    bytes as one write_volume; a second process-style attach writes into the
    same in-progress file; an exception leaves no file behind."""
    from paper_2003_12677_b200 import io
    v = io.read_volume(os.path.join(GOLDEN, "vol_sino.sptomo"))
    out = str(tmp_path / "s.sptomo")
    with io.VolumeWriter(out, v.kind, v.data.shape, center=v.center, angles=v.angles) as w:
        w.write(2, v.data[2])
        other = io.VolumeWriter.attach(w.tmp)
        other[1] = v.data[1]
        other.flush()
        w.write(0, v.data[0:1])
        assert not os.path.exists(out)
    assert open(out, "rb").read() == open(os.path.join(GOLDEN, "vol_sino.sptomo"), "rb").read()
    bad = str(tmp_path / "bad.sptomo")
    with pytest.raises(RuntimeError):
        with io.VolumeWriter(bad, io.KIND_TOMOGRAM, (2, 4, 4)) as w:
            raise RuntimeError("boom")
    assert not os.path.exists(bad) and not os.listdir(tmp_path) == []
    assert all(not f.startswith("bad.sptomo") for f in os.listdir(tmp_path))
    with pytest.raises(ValueError):
        io.write_volume(str(tmp_path / "x"), io.KIND_SINOGRAM, np.zeros((2, 3, 4)))
    with pytest.raises(ValueError):
        io.write_volume(str(tmp_path / "x"), 7, np.zeros((2, 3, 4)))


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
