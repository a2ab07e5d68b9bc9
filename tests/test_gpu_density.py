"""Device density_filter_solve (sptb_density.cu) and the density-filtered
operators against golden fixtures from the unmodified reference
(operators.py:189-236; build_operators(filter_kind="density"))."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel

pytestmark = pytest.mark.gpu

FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "density_*.npz")))
# The weights solve an ill-conditioned least-squares problem that 50 CGLS
# steps do not converge (c1: residual 121.43 of 256): the iterates depend on
# summation order at the 1e-3 level -- the unmodified reference run on the GPU
# box's CPU differs from the fixture (made in the build container) by 2.3e-3
# (scratch/density_diag.py).  The objective is well determined: the residual
# history agrees to ~1e-5.  The device solves in float64 on a complex128 build.
# north_star's 1e-4 operator bar applies to the operator given the weights.
TOL_W = 1e-2
TOL_HIST = 1e-4


@pytest.fixture(scope="module")
def sb():
    import paper_2003_12677_b200 as m
    return m


@pytest.mark.parametrize("prec", ["complex64", "complex128"])
@pytest.mark.parametrize("fname", FILES)
def test_density_filter_matches_reference(sb, fname, prec):
    d = load_golden(fname)
    g = sb.ScanGeometry(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]), angles=d["angles"],
                        n_x=int(d["n_x"]), n_y=int(d["n_y"]), center=float(d["center"]))
    k = sb.KernelSpec(family=str(d["k_family"]), width=int(d["k_width"]),
                      beta=float(d["k_beta"]), sigma=float(d["k_sigma"]))
    ops = sb.build_operators(g, k, filter_kind="density", precision=prec)
    fs = ops.filter_spec
    assert fs.kind == "density"
    assert rel(fs.weights, d["weights"]) <= TOL_W
    assert len(fs.residual_history) == len(d["residual_history"])
    np.testing.assert_allclose(fs.residual_history, d["residual_history"], rtol=TOL_HIST)
    assert abs(fs.final_residual - float(d["final_residual"])) <= TOL_HIST * float(d["final_residual"])
    assert fs.converged == bool(d["converged"])
    # The calibration and the density-filtered reconstruction inherit the
    # conditioning: the reference algorithm itself, run on the GPU box's CPU,
    # gives calib 0.0131 against the fixture's 0.0197 (c1).  The operator is
    # pinned instead with the reference's own weights and calibration:
    want = d["iradon"]
    got = sb.iradon(d["sino"], ops.csr, ops.deapo, g, weights=d["weights"], scale=float(d["calib"]))
    assert rel(got, want) <= (1e-4 if prec == "complex64" else 1e-9)
    # symmetric in p: the folded operator stays real-to-real
    w2 = fs.weights.reshape(g.n_theta, g.n_p)
    j = np.arange(g.n_p)
    np.testing.assert_allclose(w2, w2[:, (g.n_p - j) % g.n_p], rtol=0, atol=0)


def test_explicit_weights_restore_plan_state(sb):
    """iradon(..., weights=w) folds w for the call only: the bundle's own
    filtered iradon (and its calibration) is unchanged afterwards."""
    import torch
    g = sb.ScanGeometry(n_p=64, n_theta=45)
    ops = sb.build_operators(g, filter_kind="hamming")
    sino = torch.randn(2, 45, 64, device="cuda")
    before = ops.iradon(sino).cpu().numpy()
    w = np.abs(np.random.default_rng(0).standard_normal(64))
    other = sb.iradon(sino, ops.csr, ops.deapo, g, weights=w, scale=2.0).cpu().numpy()
    after = ops.iradon(sino).cpu().numpy()
    np.testing.assert_array_equal(before, after)
    assert rel(other, before) > 1e-2
