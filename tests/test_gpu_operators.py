"""Parity of the CUDA operators with the reference (golden fixtures) and the
oracle.  Tolerances: north_star's 1e-4 relative L2 per operator application
for the complex64 path; 1e-10 for the complex128 validation path."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel

pytestmark = pytest.mark.gpu

OPS_FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "ops_*.npz")))
TOL = {"complex64": 1e-4, "complex128": 1e-10}


def _geom(sb, d):
    g = sb.ScanGeometry(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]), angles=d["angles"],
                        n_x=int(d["n_x"]), n_y=int(d["n_y"]), center=float(d["center"]))
    k = sb.KernelSpec(family=str(d["k_family"]), width=int(d["k_width"]),
                      beta=float(d["k_beta"]), sigma=float(d["k_sigma"]))
    return g, k


@pytest.fixture(scope="module")
def sb():
    import paper_2003_12677_b200 as m
    return m


@pytest.fixture(scope="module", params=OPS_FILES)
def golden(request):
    return load_golden(request.param)


@pytest.mark.parametrize("prec", ["complex64", "complex128"])
def test_matrix_structure_matches_reference(sb, golden, prec):
    g, k = _geom(sb, golden)
    ops = sb.build_operators(g, k, filter_kind="none", precision=prec)
    assert ops.csr.nnz == int(golden["nnz"])
    S = ops.csr.matrix
    np.testing.assert_array_equal(S.indptr, golden["S_row_ptr"])
    np.testing.assert_array_equal(ops.csr.adjoint.indptr, golden["SH_row_ptr"])
    if "S_col_idx" in golden:
        np.testing.assert_array_equal(S.indices, golden["S_col_idx"])
        atol = 1e-7 if prec == "complex64" else 1e-14
        np.testing.assert_allclose(S.data, golden["S_vals"], rtol=0, atol=atol)
    np.testing.assert_allclose(ops.deapo.values, golden["deapo"], rtol=1e-12)


@pytest.mark.parametrize("prec", ["complex64", "complex128"])
def test_radon_adjoint_vs_reference(sb, golden, prec):
    g, k = _geom(sb, golden)
    ops = sb.build_operators(g, k, filter_kind="none", precision=prec)
    tol = TOL[prec]
    assert rel(ops.radon(golden["u"]), golden["radon_u"]) <= tol
    uc = golden["uc"] if "uc" in golden else golden["u"] + 0.5j * golden["u"].T
    assert rel(ops.radon(uc), golden["radon_uc"]) <= tol
    s = golden["s"] if "s" in golden else golden["radon_u"]
    sc = golden["sc"] if "sc" in golden else golden["radon_uc"]
    assert rel(ops.radon_adjoint(s), golden["adj_s"]) <= tol
    assert rel(ops.radon_adjoint(sc), golden["adj_sc"]) <= tol
    # real in -> real out (operators.py:166-167,185-186)
    assert not np.iscomplexobj(ops.radon(golden["u"]))


@pytest.mark.parametrize("kind", ["ramlak", "hamming", "shepplogan"])
@pytest.mark.parametrize("prec", ["complex64", "complex128"])
def test_gridrec_vs_reference(sb, golden, kind, prec):
    if f"calib_{kind}" not in golden:
        pytest.skip("fixture carries ramlak only at this size")
    g, k = _geom(sb, golden)
    ops = sb.build_operators(g, k, filter_kind=kind, precision=prec)
    tol = TOL[prec]
    assert abs(ops.calib_scale - float(golden[f"calib_{kind}"])) <= tol * abs(ops.calib_scale)
    assert rel(ops.iradon(golden["radon_u"]), golden[f"iradon_{kind}_radon_u"]) <= tol
    if f"iradon_{kind}_s" in golden:
        assert rel(ops.iradon(golden["s"]), golden[f"iradon_{kind}_s"]) <= tol
        assert rel(ops.apply_weights(golden["s"]), golden[f"apply_{kind}_s"]) <= tol
        assert rel(ops.apply_weights(golden["sc"]), golden[f"apply_{kind}_sc"]) <= tol


def test_spmv_matches_host_matrix(sb):
    d = load_golden("ops_g32.npz")
    g, k = _geom(sb, d)
    ops = sb.build_operators(g, k, filter_kind="none", precision="complex128")
    rng = np.random.default_rng(0)
    M, N = ops.csr.shape
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    import scipy.sparse as sp
    S = sp.csr_matrix((d["S_vals"], d["S_col_idx"], d["S_row_ptr"]), shape=(M, N))
    np.testing.assert_allclose(sb.spmv(ops.csr, x), S @ x, atol=1e-12)
    np.testing.assert_allclose(sb.spmv(ops.csr, y, adjoint=True), S.conj().T @ y, atol=1e-12)
    X = rng.standard_normal((N, 5)) + 1j * rng.standard_normal((N, 5))
    np.testing.assert_allclose(sb.spmm(ops.csr, X), S @ X, atol=1e-12)
    with pytest.raises(sb.ShapeMismatchError):
        sb.spmv(ops.csr, np.ones(5, dtype=complex))


def test_adjoint_identity_and_linearity(sb):
    """criterion 1 (test_acceptance.py:35-49) and test_operators.py:248-270."""
    geom = sb.ScanGeometry(n_p=64, n_theta=45)
    ops = sb.build_operators(geom, filter_kind="none", precision="complex128")
    rng = np.random.default_rng(1)
    for _ in range(5):
        u = rng.standard_normal(geom.grid_shape) + 1j * rng.standard_normal(geom.grid_shape)
        s = rng.standard_normal(geom.sino_shape) + 1j * rng.standard_normal(geom.sino_shape)
        lhs = np.vdot(s, ops.radon(u))
        rhs = np.vdot(ops.radon_adjoint(s), u)
        assert abs(lhs - rhs) <= 1e-8 * abs(lhs)
        v = rng.standard_normal(geom.grid_shape)
        a, b = rng.standard_normal(2)
        assert rel(ops.radon(a * u + b * v), a * ops.radon(u) + b * ops.radon(v)) <= 1e-10


def test_real_leakage_and_pairing(sb):
    """test_operators.py:273-277 and criterion 8 (pairing <= 1e-5)."""
    from oracle import shepp_logan
    geom = sb.ScanGeometry(n_p=64, n_theta=40)
    ops = sb.build_operators(geom, filter_kind="ramlak")
    u = shepp_logan(64)[0]
    s = ops.radon(u.astype(complex))
    assert np.linalg.norm(s.imag) <= 1e-6 * np.linalg.norm(s.real)
    rng = np.random.default_rng(2)
    sa, sb_ = rng.standard_normal((2,) + geom.sino_shape)
    ra, rb = ops.iradon(sa), ops.iradon(sb_)
    rp = ops.iradon(sa + 1j * sb_)
    assert rel(rp.real, ra) <= 1e-5 and rel(rp.imag, rb) <= 1e-5


@pytest.mark.parametrize("n", [1, 2, 3, 8, 65])
def test_batched_device_tensors(sb, n):
    """(n, ...) stacks of real slices on the device == per-slice host calls."""
    import torch
    from oracle import OGeom, build_oracle_ops
    geom = sb.ScanGeometry(n_p=32, n_theta=20)
    ops = sb.build_operators(geom, filter_kind="ramlak", max_batch=32)
    oops = build_oracle_ops(OGeom(32, 20), kind="ramlak")
    rng = np.random.default_rng(n)
    u = rng.standard_normal((n,) + geom.grid_shape)
    sd = ops.radon(torch.tensor(u, dtype=torch.float32, device="cuda"))
    rd = ops.iradon(sd)
    torch.cuda.synchronize()
    want_s = np.stack([oops.radon(x) for x in u])
    want_r = np.stack([oops.iradon(x) for x in want_s])
    assert sd.shape == (n,) + geom.sino_shape and sd.dtype == torch.float32
    assert rel(sd.cpu().numpy(), want_s) <= 1e-4
    assert rel(rd.cpu().numpy(), want_r) <= 1e-4
    # host f64 batch path through the C ABI staging
    assert rel(ops.radon(u), want_s) <= 1e-4


def test_config1_operators(sb):
    """Config 1: 256^2 phantom, 180 angles: R, R^T, gridrec vs reference <= 1e-4."""
    d = load_golden("ops_c1.npz")
    g, k = _geom(sb, d)
    ops_n = sb.build_operators(g, k, filter_kind="none")
    ops_r = sb.build_operators(g, k, filter_kind="ramlak")
    assert rel(ops_n.radon(d["u"]), d["radon_u"]) <= 1e-4
    assert rel(ops_n.radon_adjoint(d["radon_u"]), d["adj_s"]) <= 1e-4
    assert rel(ops_r.iradon(d["radon_u"]), d["iradon_ramlak_radon_u"]) <= 1e-4


def test_shape_errors(sb):
    ops = sb.build_operators(sb.ScanGeometry(n_p=16, n_theta=6), filter_kind="none")
    with pytest.raises(sb.ShapeMismatchError):
        ops.radon(np.zeros((8, 8)))
    with pytest.raises(sb.ShapeMismatchError):
        ops.iradon(np.zeros((6, 8)))


def test_zero_inputs(sb):
    ops = sb.build_operators(sb.ScanGeometry(n_p=16, n_theta=6))
    np.testing.assert_array_equal(ops.radon(np.zeros((16, 16))), 0.0)
    np.testing.assert_array_equal(ops.iradon(np.zeros((6, 16))), 0.0)


def test_near_zero_deapodization_raises(sb):
    # KB width 5, beta = 3 pi / 4: FT(K) has its first zero exactly at nu = 1/4,
    # i.e. on the grid column n_x/2 + n_x/4 inside the support disk
    import math
    with pytest.raises(sb.NearZeroDenominatorError):
        sb.build_operators(sb.ScanGeometry(n_p=16, n_theta=4),
                           kernel=sb.KernelSpec(width=5, beta=0.75 * math.pi))


def test_precondition_matches_reference(sb):
    """precondition_apply(pre, sino) with the reference's signature (no ops:
    a cached device plan for the sinogram's shape), TomoOperators.precondition
    and preconditioner(kind) against the unmodified reference
    (operators.py:85-121,262-290); complex128 plans for NumPy input, a
    complex64 plan for float32 device tensors."""
    import torch
    d = load_golden("precond_g32.npz")
    geom = sb.ScanGeometry(n_p=32, n_theta=20)
    ops = sb.build_operators(geom, filter_kind="ramlak")
    for kind in ("hamming", "ramlak", "none"):
        pre = ops.preconditioner(kind)
        np.testing.assert_array_equal(pre.weights, d[f"pre_{kind}_w"])
        assert rel(sb.precondition_apply(pre, d["s"]), d[f"pre_{kind}_s"]) <= 1e-12
        out = sb.precondition_apply(pre, d["sc"])
        assert np.iscomplexobj(out) and rel(out, d[f"pre_{kind}_sc"]) <= 1e-12
        # through a complex64 bundle: that plan's precision
        assert rel(sb.precondition_apply(pre, d["s"], ops), d[f"pre_{kind}_s"]) <= 1e-6
    ops_h = sb.build_operators(geom, filter_kind="hamming")
    assert rel(ops_h.precondition(d["s"]), d["ops_hamming_precondition_s"]) <= 1e-6
    ops_h64 = sb.build_operators(geom, filter_kind="hamming", precision="complex128")
    assert rel(ops_h64.precondition(d["s"]), d["ops_hamming_precondition_s"]) <= 1e-12
    pre = sb.Preconditioner(weights=d["wfull"])
    assert rel(sb.precondition_apply(pre, d["sc"]), d["pre_full_sc"]) <= 1e-12
    hpre = ops.preconditioner("hamming")
    assert rel(sb.precondition_apply(hpre, d["s7"]), d["pre_hamming_s7"]) <= 1e-12
    row = sb.precondition_apply(hpre, d["s7"][3])
    assert row.shape == (32,) and rel(row, d["pre_hamming_row"]) <= 1e-12
    t = torch.tensor(d["s"], dtype=torch.float32, device="cuda")
    out = sb.precondition_apply(hpre, t)
    assert out.is_cuda and out.dtype == torch.float32
    assert rel(out.cpu().numpy(), d["pre_hamming_s"]) <= 1e-5
    with pytest.raises(sb.ShapeMismatchError):
        sb.precondition_apply(hpre, np.zeros((20, 31)))


@pytest.mark.parametrize("prec,tol", [("complex128", 1e-10), ("complex64", 1e-4)])
def test_threshold_build_matches_reference(sb, prec, tol):
    """threshold > 0 (gridding.py:159-163): S pruned on |v|, the filtered
    matrix on its weighted values |w v| -- structure identical to the
    reference's, and the operators and calibration built on them."""
    d = load_golden("threshold_g32.npz")
    ops = sb.build_operators(sb.ScanGeometry(n_p=32, n_theta=20), filter_kind="ramlak",
                             threshold=0.05, precision=prec)
    for tag, m in (("S", ops.csr), ("SF", ops.csr_filtered)):
        np.testing.assert_array_equal(m.row_ptr, d[f"{tag}_row_ptr"])
        np.testing.assert_array_equal(m.col_idx, d[f"{tag}_col"])
        assert rel(m.vals, d[f"{tag}_vals"]) <= min(tol, 1e-6)
        assert m.nnz == len(d[f"{tag}_vals"])
    assert abs(ops.calib_scale - float(d["calib"])) <= tol * abs(float(d["calib"]))
    assert rel(ops.radon(d["u"]), d["radon_u"]) <= tol
    assert rel(ops.radon_adjoint(d["s"]), d["adj_s"]) <= tol
    assert rel(ops.iradon(d["s"]), d["iradon_s"]) <= tol


def test_production_batch_kernels_on_golden_geometries(sb, golden):
    """The 32-vector launch (64 real slices) takes the production S kernel
    (length-sorted row pairs, long-row CTAs) and the batched FFT passes on
    every golden geometry -- odd n_p, off-centre, rectangular grid, width-5
    and Gaussian kernels, custom angles, config 1: each slice of the batch
    matches the reference's radon / radon_adjoint / iradon of that slice."""
    import torch
    g, k = _geom(sb, golden)
    has_s = "s" in golden
    s_in = golden["s"] if has_s else golden["radon_u"]
    key = "s" if has_s else "radon_u"
    kind = next((kk for kk in ("ramlak", "hamming") if f"iradon_{kk}_{key}" in golden), None)
    sc = torch.linspace(0.5, 1.5, 64, dtype=torch.float64)[:, None, None]
    sino = (torch.tensor(s_in)[None] * sc).to(torch.float32).cuda().contiguous()
    img = (torch.tensor(golden["u"])[None] * sc).to(torch.float32).cuda().contiguous()
    ops_n = sb.build_operators(g, k, filter_kind="none", max_batch=32)
    ra = ops_n.radon_adjoint(sino).cpu().numpy()
    rs = ops_n.radon(img).cpu().numpy()
    rec = None
    if kind:
        ops = sb.build_operators(g, k, filter_kind=kind, max_batch=32)
        rec = ops.iradon(sino).cpu().numpy()
    for z in (0, 1, 17, 62, 63):
        f = float(sc[z])
        assert rel(ra[z], f * golden["adj_s"]) <= 1e-4, z
        assert rel(rs[z], f * golden["radon_u"]) <= 1e-4, z
        if kind:
            assert rel(rec[z], f * golden[f"iradon_{kind}_{key}"]) <= 1e-4, z
