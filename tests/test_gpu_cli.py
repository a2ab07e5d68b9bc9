"""``python -m paper_2003_12677_b200 recon`` against the reference CLI
(cli.py:111-161, golden fixture made by running the unmodified reference's
``sptomo phantom`` / ``recon``; tests/golden/make_golden.py cli_case):
the same input volume, flags and exit codes, results within the solver
parity bars (complex64 production path: 1e-3 for FBP / SIRT; CGLS within
its emulated-fp32 floor, test_gpu_solvers.py)."""

import json
import os

import numpy as np
import pytest

from conftest import load_golden, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return load_golden("cli_g32.npz")


def _write(tmp_path, name, raw):
    p = str(tmp_path / name)
    with open(p, "wb") as fh:
        fh.write(raw.tobytes())
    return p


@pytest.mark.parametrize("algo,iters,tol", [("fbp", 1, 1e-3), ("sirt", 4, 1e-3), ("cgls", 3, 5e-3)])
def test_recon_matches_reference_cli(tmp_path, gold, algo, iters, tol):
    from paper_2003_12677_b200 import io
    from paper_2003_12677_b200.cli import EXIT_OK, main
    sino = _write(tmp_path, "sino.spt", gold["sino_bytes"])
    out, met = str(tmp_path / "rec.spt"), str(tmp_path / "met.json")
    assert main(["recon", "--in", sino, "--out", out, "--algo", algo, "--iters", str(iters),
                 "--metrics-out", met]) == EXIT_OK
    v = io.read_volume(out)
    assert v.kind == io.KIND_TOMOGRAM and v.data.shape == (3, 32, 32) and v.angles is None
    assert rel(v.data, gold[f"rec_{algo}"]) <= tol
    rec = json.load(open(met))[0]
    assert rec["algo"] == algo and rec["iters"] == iters and rec["snr_db"] is None
    np.testing.assert_allclose(rec["residual_history"], gold[f"hist_{algo}"], rtol=max(tol, 1e-3))
    assert not [f for f in os.listdir(tmp_path) if ".tmp" in f]


def test_recon_intensity_volume(tmp_path, gold):
    from paper_2003_12677_b200 import io
    from paper_2003_12677_b200.cli import EXIT_OK, main
    inten = _write(tmp_path, "int.spt", gold["int_bytes"])
    out = str(tmp_path / "rec.spt")
    assert main(["recon", "--in", inten, "--out", out, "--algo", "fbp"]) == EXIT_OK
    assert rel(io.read_volume(out).data, gold["rec_int_fbp"]) <= 1e-3


def test_recon_errors(tmp_path, gold, capsys):
    from paper_2003_12677_b200 import io
    from paper_2003_12677_b200.cli import EXIT_ERROR, EXIT_OK, main
    missing = str(tmp_path / "nope.spt")
    assert main(["recon", "--in", missing, "--out", str(tmp_path / "r.spt")]) == EXIT_ERROR
    assert missing in capsys.readouterr().err
    sino = _write(tmp_path, "sino.spt", gold["sino_bytes"])
    out = str(tmp_path / "rec.spt")
    assert main(["recon", "--in", sino, "--out", out]) == EXIT_OK
    assert main(["recon", "--in", out, "--out", str(tmp_path / "r2.spt")]) == EXIT_ERROR
    assert "tomogram" in capsys.readouterr().err
    # a centre override changes the reconstruction (cli.py:138-142)
    out_c = str(tmp_path / "rec_c.spt")
    assert main(["recon", "--in", sino, "--out", out_c, "--center", "14.5"]) == EXIT_OK
    assert not np.allclose(io.read_volume(out).data, io.read_volume(out_c).data)


def test_recon_uses_cache_dir(tmp_path, gold):
    from paper_2003_12677_b200.cli import EXIT_OK, main
    sino = _write(tmp_path, "sino.spt", gold["sino_bytes"])
    cache = str(tmp_path / "cache")
    os.makedirs(cache)
    assert main(["recon", "--in", sino, "--out", str(tmp_path / "r.spt"), "--cache", cache]) == EXIT_OK
    files = os.listdir(cache)
    assert sum(f.endswith(".sgcsr") for f in files) == 2          # S and S diag(w), ramlak
    assert sum(f.endswith(".meta.json") for f in files) == 1      # its calibration
