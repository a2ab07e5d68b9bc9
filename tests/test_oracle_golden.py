"""Pin the CPU oracle against golden vectors from the unmodified reference."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_geom, load_golden, rel
from oracle import (build_gridding, build_oracle_ops, deapodization, o_solve,
                    op_apply_weights, filter_weights, OGeom, OracleOps)

OPS_FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "ops_*.npz")))


@pytest.fixture(scope="module", params=OPS_FILES)
def case(request):
    d = load_golden(request.param)
    g, k = golden_geom(d)
    return d, g, k, build_oracle_ops(g, k, "none")


def test_matrix_structure(case):
    d, g, k, ops = case
    assert ops.grid.nnz == int(d["nnz"])
    np.testing.assert_array_equal(ops.grid.S.indptr, d["S_row_ptr"])
    np.testing.assert_array_equal(ops.grid.SH.indptr, d["SH_row_ptr"])
    if "S_col_idx" in d:
        np.testing.assert_array_equal(ops.grid.S.indices, d["S_col_idx"])
        np.testing.assert_array_equal(ops.grid.SH.indices, d["SH_col_idx"])
        np.testing.assert_allclose(ops.grid.S.data, d["S_vals"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(ops.grid.SH.data, d["SH_vals"], rtol=0, atol=1e-15)
    assert abs(np.abs(ops.grid.S.data).sum() - float(d["S_abs_sum"])) <= 1e-9 * float(d["S_abs_sum"])


def test_deapodization(case):
    d, g, k, ops = case
    np.testing.assert_allclose(ops.deapo, d["deapo"], rtol=1e-13, atol=0)


def test_radon_and_adjoint(case):
    d, g, k, ops = case
    assert rel(ops.radon(d["u"]), d["radon_u"]) <= 1e-12
    assert rel(ops.radon(_uc(d)), d["radon_uc"]) <= 1e-12
    assert rel(ops.radon_adjoint(_s(d, ops)), d["adj_s"]) <= 1e-12
    assert rel(ops.radon_adjoint(_sc(d, ops)), d["adj_sc"]) <= 1e-12


def _uc(d):
    return d["uc"] if "uc" in d else d["u"] + 0.5j * d["u"].T


def _s(d, ops):
    return d["s"] if "s" in d else ops.radon(d["u"])


def _sc(d, ops):
    return d["sc"] if "sc" in d else ops.radon(_uc(d))


@pytest.mark.parametrize("kind", ["ramlak", "hamming", "shepplogan"])
def test_filtered_iradon_and_calibration(case, kind):
    d, g, k, _ = case
    if f"calib_{kind}" not in d:
        pytest.skip("fixture carries ramlak only at this size")
    fops = build_oracle_ops(g, k, kind)
    assert abs(fops.calib - float(d[f"calib_{kind}"])) <= 1e-12 * abs(fops.calib)
    assert rel(fops.iradon(d["radon_u"]), d[f"iradon_{kind}_radon_u"]) <= 1e-11
    if f"iradon_{kind}_s" in d:
        assert rel(fops.iradon(d["s"]), d[f"iradon_{kind}_s"]) <= 1e-11
        assert rel(fops.apply_weights(d["s"]), d[f"apply_{kind}_s"]) <= 1e-13
        assert rel(fops.apply_weights(d["sc"]), d[f"apply_{kind}_sc"]) <= 1e-13


@pytest.fixture(scope="module")
def sol():
    return load_golden("solvers_g32.npz")


@pytest.mark.parametrize("algo,iters", [("fbp", 1), ("sirt", 8), ("cgls", 8), ("tv", 5)])
def test_solvers_match_reference(sol, algo, iters):
    kind = {"fbp": "ramlak", "sirt": "hamming", "cgls": "none", "tv": "none"}[algo]
    ops = build_oracle_ops(OGeom(n_p=32, n_theta=20), kind=kind)
    sa, sb = sol[f"{algo}_sino_a"], sol[f"{algo}_sino_b"]
    rp, rep_p = o_solve(sa + 1j * sb, ops, algo, max_iter=iters)
    ra, rep_a = o_solve(sa, ops, algo, max_iter=iters)
    assert rel(rp, sol[f"{algo}_rec_pair"]) <= 1e-10
    assert rel(ra, sol[f"{algo}_rec_a"]) <= 1e-10
    np.testing.assert_allclose(rep_p.history, sol[f"{algo}_hist_pair"], rtol=1e-10)
    np.testing.assert_allclose(rep_a.history, sol[f"{algo}_hist_a"], rtol=1e-10)
    assert rep_p.iterations == int(sol[f"{algo}_iters_pair"])


def test_solver_variants(sol):
    ops = build_oracle_ops(OGeom(n_p=32, n_theta=20), kind="hamming")
    sa = sol["sirt_sino_a"]
    for tag, kw in (("sirt_nobb", dict(max_iter=6, bb=False)),
                    ("sirt_nonneg", dict(max_iter=6, nonneg=True)),
                    ("sirt_tol", dict(max_iter=50, tol=0.05))):
        r, rep = o_solve(sa, ops, "sirt", **kw)
        assert rel(r, sol[f"{tag}_rec"]) <= 1e-10, tag
        assert rep.iterations == int(sol[f"{tag}_iters"]), tag
        np.testing.assert_allclose(rep.history, sol[f"{tag}_hist"], rtol=1e-10)
    opn = build_oracle_ops(OGeom(n_p=32, n_theta=20), kind="none")
    r, rep = o_solve(sol["tv_sino_a"], opn, "tv", max_iter=3, mu=0.5)
    assert rel(r, sol["tv_mu_rec"]) <= 1e-10


def test_precondition_matches_reference():
    """precondition_apply (operators.py:108-121) for radial / per-sample
    weights, real / complex input, other angle counts and one detector row."""
    from oracle.tomo import op_precondition
    d = load_golden("precond_g32.npz")
    for kind in ("hamming", "ramlak", "none"):
        w = d[f"pre_{kind}_w"]
        assert rel(op_precondition(d["s"], w), d[f"pre_{kind}_s"]) <= 1e-13
        assert rel(op_precondition(d["sc"], w), d[f"pre_{kind}_sc"]) <= 1e-13
    assert rel(op_precondition(d["sc"], d["wfull"]), d["pre_full_sc"]) <= 1e-13
    assert rel(op_precondition(d["s7"], d["pre_hamming_w"]), d["pre_hamming_s7"]) <= 1e-13


CGS_TAGS = [("", dict(max_iter=8)), ("_nonneg", dict(max_iter=6, nonneg=True)),
            ("_tol", dict(max_iter=40, tol=0.02))]


@pytest.mark.parametrize("kind", ["none", "hamming"])
@pytest.mark.parametrize("tag,kw", CGS_TAGS)
def test_cgs_mode_matches_reference(kind, tag, kw):
    """solve_cgls with cgs_mode=True (solvers.py:247-248,262-305)."""
    d = load_golden("solvers_cgs_g32.npz")
    ops = build_oracle_ops(OGeom(n_p=32, n_theta=20), kind=kind)
    sa, sb = d[f"{kind}_sino_a"], d[f"{kind}_sino_b"]
    for sino, key in ((sa + 1j * sb, "pair"), (sa, "a")):
        r, rep = o_solve(sino, ops, "cgls", cgs_mode=True, **kw)
        assert rel(r, d[f"{kind}{tag}_rec_{key}"]) <= 1e-10
        np.testing.assert_allclose(rep.history, d[f"{kind}{tag}_hist_{key}"], rtol=1e-10)
        assert rep.converged == bool(d[f"{kind}{tag}_conv_{key}"])


DENSITY_FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "density_*.npz")))


@pytest.mark.parametrize("fname", DENSITY_FILES)
def test_density_weights(fname):
    """density_filter_solve (operators.py:189-236) and the density-filtered
    gridrec built on it (build_operators(filter_kind="density"))."""
    from oracle import density_weights
    d = load_golden(fname)
    g, k = golden_geom(d)
    w, hist, conv, fin = density_weights(build_gridding(g, k), g)
    # ill-conditioned (see tests/test_gpu_density.py): exact in the container
    # that made the fixture, ~2e-3 on other CPUs; the objective agrees to 1e-5
    assert rel(w, d["weights"]) <= 1e-2
    np.testing.assert_allclose(hist, d["residual_history"], rtol=1e-4)
    assert conv == bool(d["converged"])
    assert abs(fin - float(d["final_residual"])) <= 1e-4 * max(1.0, float(d["final_residual"]))
    # calib / filtered reconstruction inherit the conditioning (the reference
    # run on another CPU gives calib 0.0131 vs 0.0197 at c1): pinned on the
    # container that made the fixture only through the objective above
