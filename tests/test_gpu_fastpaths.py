"""The production fast paths against the general ones and the CPU oracle.

Each fast path of the hot loop has a general fallback that the parity tests
(test_gpu_operators.py) also exercise at small batch sizes.  These tests run
both on the same batched inputs, at sizes where the fast path is the one
taken (n_p a power of two >= 128, batch a multiple of 4 complex vectors):

* fused pack + FFT1 + permute / gather + IFFT1 + unpack (sptb_fft.cu):
  Stockham kernel for n_p <= 256, register radix-16 kernel for n_p >= 512;
* fused inverse FFT2 (y pass in place, x pass + deapodization + unpack) vs
  cuFFT's 2-D plan + unpack (SPTB_NO_FUSED_FFT2);
* S^H through the TMA-staged slot kernel vs the LDGSTS slot kernel
  (sptb_patch.cu; SPTB_NO_TMA selects the latter per call);
* the oracle (reference algorithm restated on the CPU) on a few slices.

Tolerance: north_star's 1e-4 relative L2 per operator application (complex64).
"""

import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2003_12677_b200 as m
    return m


def _env(name, value):
    """Set an SPTB_* path switch for the block (the library reads the switches
    once; sptb_reload_switches re-reads them)."""
    from paper_2003_12677_b200 import _lib

    class _E:
        def __enter__(self):
            self.old = os.environ.get(name)
            os.environ[name] = value
            _lib.lib.sptb_reload_switches()

        def __exit__(self, *a):
            if self.old is None:
                os.environ.pop(name, None)
            else:
                os.environ[name] = self.old
            _lib.lib.sptb_reload_switches()
    return _E()


def _ops(sb, n, T, kind="ramlak"):
    return sb.build_operators(sb.ScanGeometry(n_p=n, n_theta=T), filter_kind=kind, max_batch=8)


@pytest.mark.parametrize("n,T", [(128, 45), (256, 90), (512, 60), (1024, 40), (2048, 12), (4096, 6)])
def test_fused_fft1_matches_cufft_path(sb, n, T):
    import torch
    ops = _ops(sb, n, T)
    g = torch.Generator(device="cuda").manual_seed(n)
    sino = torch.randn(13, T, n, device="cuda", generator=g)   # odd stack: 7 units, tail unpaired
    img = torch.randn(13, n, n, device="cuda", generator=g)
    rec_fast, sin_fast = ops.iradon(sino), ops.radon(img)
    with _env("SPTB_NO_FUSED_FFT1", "1"):
        rec_ref, sin_ref = ops.iradon(sino), ops.radon(img)
    with _env("SPTB_FFT1_FWD_ROWS", "1"):  # row-FFT kernel instead of the TMA column pass
        rec_rows = ops.iradon(sino)
        with _env("SPTB_FFT1_NO_BULK", "1"):  # ... with per-lane loads
            rec_lanes = ops.iradon(sino)
    with _env("SPTB_FFT1_INV_GATHER", "1"):  # S^H in patch order + gathering inverse FFT1
        sin_gather = ops.radon(img)
    torch.cuda.synchronize()
    assert rel(sin_fast.cpu().numpy(), sin_gather.cpu().numpy()) < 1e-6
    assert rel(rec_fast.cpu().numpy(), rec_ref.cpu().numpy()) < 1e-5
    assert rel(rec_fast.cpu().numpy(), rec_rows.cpu().numpy()) < 1e-6
    assert rel(rec_fast.cpu().numpy(), rec_lanes.cpu().numpy()) < 1e-6
    assert rel(sin_fast.cpu().numpy(), sin_ref.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("n,T,nx,ny", [(512, 60, None, None), (1024, 40, None, None), (2048, 12, None, None),
                                       (4096, 6, None, None), (512, 45, 1024, 512), (1024, 30, 512, 2048)])
def test_fused_fft2_unpack_matches_cufft_path(sb, n, T, nx, ny):
    """iradon's y pass + x pass/deapodization/unpack and radon's pack/x pass +
    y pass vs cuFFT + pack/unpack (square and rectangular grids, odd stack:
    the last pair has no partner)."""
    import torch
    ops = sb.build_operators(sb.ScanGeometry(n_p=n, n_theta=T, n_x=nx, n_y=ny), filter_kind="ramlak",
                             max_batch=8)
    g = torch.Generator(device="cuda").manual_seed(n + T)
    sino = torch.randn(13, T, n, device="cuda", generator=g)
    img = torch.randn(13, ops.geom.n_y, ops.geom.n_x, device="cuda", generator=g)
    fast, fast_s = ops.iradon(sino), ops.radon(img)
    with _env("SPTB_NO_FUSED_FFT2", "1"):
        ref, ref_s = ops.iradon(sino), ops.radon(img)
    torch.cuda.synchronize()
    assert fast.shape == ref.shape
    assert rel(fast.cpu().numpy(), ref.cpu().numpy()) < 1e-5
    assert rel(fast_s.cpu().numpy(), ref_s.cpu().numpy()) < 1e-5


def test_fused_fft1_stockham_variant(sb):
    """n_p >= 512: the forward runs the register radix-16 kernel by default
    (the Stockham kernel below 512); both give the same iradon."""
    import torch
    ops = _ops(sb, 512, 30)
    sino = torch.randn(8, 30, 512, device="cuda")
    a = ops.iradon(sino)
    with _env("SPTB_FFT1_STOCKHAM", "1"):
        b = ops.iradon(sino)
    torch.cuda.synchronize()
    assert rel(a.cpu().numpy(), b.cpu().numpy()) < 1e-5


def test_sh_tma_matches_ldgsts_kernel(sb):
    import torch
    ops = _ops(sb, 256, 90, "none")
    img = torch.randn(16, 256, 256, device="cuda")
    a = ops.radon(img)
    with _env("SPTB_NO_TMA", "1"):
        b = ops.radon(img)
    torch.cuda.synchronize()
    assert rel(a.cpu().numpy(), b.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("n,T", [(256, 180), (512, 120)])
def test_fast_paths_vs_oracle(sb, n, T):
    import torch
    from oracle import OGeom, build_oracle_ops, shepp_logan
    ops = _ops(sb, n, T)
    oops = build_oracle_ops(OGeom(n_p=n, n_theta=T), kind="ramlak")
    u = shepp_logan(n, 8)
    sino = ops.radon(torch.tensor(u, dtype=torch.float32, device="cuda"))
    rec = ops.iradon(sino)
    torch.cuda.synchronize()
    s_np, r_np = sino.cpu().numpy(), rec.cpu().numpy()
    for i in (0, 3, 7):
        want_s = oops.radon(u[i])
        assert rel(s_np[i], want_s) < 1e-4
        assert rel(r_np[i], oops.iradon(want_s)) < 1e-4


def test_host_pipelined_io_matches_device(sb):
    """Host buffers go through the chunked H2D / compute / D2H pipeline."""
    import torch
    ops = _ops(sb, 256, 90)
    sino = torch.randn(22, 90, 256)
    dev = ops.iradon(sino.cuda()).cpu()
    host = ops.iradon(sino.numpy())
    assert rel(np.asarray(host), dev.numpy()) < 1e-6


@pytest.mark.parametrize("algo,kind", [("sirt", "hamming"), ("cgls", "none"), ("tv", "none")])
def test_solvers_fused_fft2_matches_cufft(sb, algo, kind):
    """Solver grids (n = 512) go through the in-place fused FFT2 (TMA column
    pass + bulk-copied row pass); the same solve with cuFFT's 2-D plan must
    agree to the solver tolerance (1e-3) and run the same iterations."""
    from oracle import shepp_logan
    from paper_2003_12677_b200.solvers import solve_batch
    ops = _ops(sb, 512, 96, kind)
    sino = ops.radon(shepp_logan(512, 4).astype(np.float32))
    cfg = sb.SolverConfig(algorithm=algo, max_iter=6)
    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    with _env("SPTB_NO_FUSED_FFT2", "1"):
        rec2, rep2, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    assert [r.iterations_run for r in rep] == [r.iterations_run for r in rep2]
    assert rel(np.asarray(rec), np.asarray(rec2)) < 1e-3
    if algo == "sirt":  # update + x pass fused vs OpSirtUpdate and the separate FFT2
        with _env("SPTB_SIRT_UNFUSED", "1"):
            rec3, rep3, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
        assert [r.iterations_run for r in rep] == [r.iterations_run for r in rep3]
        assert rel(np.asarray(rec), np.asarray(rec3)) < 1e-4


@pytest.mark.parametrize("nslices", [1, 5, 9, 64])
def test_partial_batches_through_persistent_passes(sb, nslices):
    """Stacks that leave whole 4-unit groups / planes of a 32-unit batch empty:
    the persistent passes still complete every buffer's mbarrier phase (a
    skipped phase would hang or read stale data) and zero the empty planes."""
    import torch
    ops = sb.build_operators(sb.ScanGeometry(n_p=512, n_theta=48), filter_kind="ramlak", max_batch=32)
    g = torch.Generator(device="cuda").manual_seed(nslices)
    sino = torch.randn(nslices, 48, 512, device="cuda", generator=g)
    img = torch.randn(nslices, 512, 512, device="cuda", generator=g)
    fast, fast_s = ops.iradon(sino), ops.radon(img)
    with _env("SPTB_FFT2_NO_PERSIST", "1"):
        ref, ref_s = ops.iradon(sino), ops.radon(img)
    torch.cuda.synchronize()
    assert rel(fast.cpu().numpy(), ref.cpu().numpy()) < 1e-6
    assert rel(fast_s.cpu().numpy(), ref_s.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("n,T,nx,ny", [(4096, 6, None, None), (1024, 24, 512, 2048), (512, 45, 1024, 512)])
def test_sirt_fused_passes_other_grids(sb, n, T, nx, ny):
    """The fused SIRT x passes at 4096-wide rows (1024-thread CTAs) and on
    rectangular grids vs the unfused element passes + FFT2."""
    import torch
    from paper_2003_12677_b200.solvers import solve_batch
    ops = sb.build_operators(sb.ScanGeometry(n_p=n, n_theta=T, n_x=nx, n_y=ny), filter_kind="hamming",
                             max_batch=4)
    g = torch.Generator(device="cuda").manual_seed(n + T)
    img = torch.rand(4, ops.geom.n_y, ops.geom.n_x, device="cuda", generator=g)
    sino = ops.radon(img)
    cfg = sb.SolverConfig(algorithm="sirt", max_iter=4)
    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    with _env("SPTB_SIRT_UNFUSED", "1"):
        rec2, rep2, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    assert [r.iterations_run for r in rep] == [r.iterations_run for r in rep2]
    assert rel(np.asarray(rec.cpu() if hasattr(rec, "cpu") else rec),
               np.asarray(rec2.cpu() if hasattr(rec2, "cpu") else rec2)) < 1e-4


@pytest.mark.parametrize("n,T,nx,ny,inner,nonneg", [
    (512, 96, None, None, 2, False), (512, 96, None, None, 3, True), (512, 96, None, None, 1, False),
    (4096, 6, None, None, 2, False), (1024, 24, 512, 2048, 2, True), (512, 45, 1024, 512, 2, False)])
def test_tv_fused_passes_match_unfused(sb, n, T, nx, ny, inner, nonneg):
    """The TV element passes fused into the FFT2 x passes (k_tv_rowfft: IFFT_x
    + OpTvS + FFT_x, IFFT_x + OpTvStepS, OpTvS + FFT_x, OpTvShrink + FFT_x) vs
    the separate element passes and FFT2 (SPTB_XPASS_UNFUSED), both against the
    complex128 build: same iterations, and the fused result as close to the
    complex128 one as the unfused (max(1e-4, 3x its deviation): complex64 TV
    moves by ~1e-3 under rounding-level changes where the shrink threshold
    cuts many pixels) -- including 1 and 3 inner steps, the nonneg
    projection, 4096-wide rows and rectangular grids."""
    import torch
    from oracle import shepp_logan
    from paper_2003_12677_b200.solvers import solve_batch
    geom = sb.ScanGeometry(n_p=n, n_theta=T, n_x=nx, n_y=ny)
    ops = sb.build_operators(geom, filter_kind="none", max_batch=4)
    if nx is None:
        img = torch.from_numpy(shepp_logan(n, 8).astype(np.float32)).cuda()
        img = img * torch.linspace(0.5, 1.5, 8, device="cuda")[:, None, None]
    else:
        g = torch.Generator(device="cuda").manual_seed(n + T + inner)
        img = torch.rand(8, ops.geom.n_y, ops.geom.n_x, device="cuda", generator=g)
    sino = ops.radon(img)
    cfg = sb.SolverConfig(algorithm="tv", max_iter=4, tv_inner_iter=inner, nonneg=nonneg)

    def host(r):
        return np.asarray(r.cpu() if hasattr(r, "cpu") else r, dtype=np.float64)

    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    with _env("SPTB_XPASS_UNFUSED", "1"):
        rec2, rep2, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    ops64 = sb.build_operators(geom, filter_kind="none", max_batch=4, precision="complex128")
    rec3, rep3, _ = solve_batch(sino.double().cpu().numpy(), ops64, cfg, raise_on_failure=False)
    its = [[r.iterations_run for r in x] for x in (rep, rep2, rep3)]
    assert its[0] == its[1] == its[2] == [4] * len(rep), (its, [r.__dict__ for r in rep])
    a, b, c = host(rec), host(rec2), host(rec3)
    assert np.isfinite(a).all()
    ea, eb = rel(a, c), rel(b, c)
    print(f"fused {ea:.2e} unfused {eb:.2e} from complex128")
    assert ea <= max(1e-4, 3 * eb), (ea, eb)


@pytest.mark.parametrize("n,T,nx,ny,nonneg", [
    (512, 96, None, None, False), (512, 96, None, None, True), (4096, 6, None, None, False),
    (1024, 24, 512, 2048, False), (512, 45, 1024, 512, True)])
def test_cgls_fused_passes_match_unfused(sb, n, T, nx, ny, nonneg):
    """CGLS with its element passes fused into the FFT2 x passes (IFFT_x +
    OpCglsInit + FFT_x, IFFT_x + <s,s>, OpCglsTail + FFT_x) vs the separate
    passes (SPTB_XPASS_UNFUSED), both against the complex128 build."""
    import torch
    from oracle import shepp_logan
    from paper_2003_12677_b200.solvers import solve_batch
    geom = sb.ScanGeometry(n_p=n, n_theta=T, n_x=nx, n_y=ny)
    ops = sb.build_operators(geom, filter_kind="none", max_batch=4)
    if nx is None:
        img = torch.from_numpy(shepp_logan(n, 8).astype(np.float32)).cuda()
    else:
        g = torch.Generator(device="cuda").manual_seed(n + T)
        img = torch.rand(8, ops.geom.n_y, ops.geom.n_x, device="cuda", generator=g)
    sino = ops.radon(img)
    cfg = sb.SolverConfig(algorithm="cgls", max_iter=8, nonneg=nonneg)

    def host(r):
        return np.asarray(r.cpu() if hasattr(r, "cpu") else r, dtype=np.float64)

    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    with _env("SPTB_XPASS_UNFUSED", "1"):
        rec2, rep2, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    ops64 = sb.build_operators(geom, filter_kind="none", max_batch=4, precision="complex128")
    rec3, rep3, _ = solve_batch(sino.double().cpu().numpy(), ops64, cfg, raise_on_failure=False)
    its = [[r.iterations_run for r in x] for x in (rep, rep2, rep3)]
    assert its[0] == its[1] == its[2], its
    a, b, c = host(rec), host(rec2), host(rec3)
    assert np.isfinite(a).all()
    ea, eb = rel(a, c), rel(b, c)
    print(f"fused {ea:.2e} unfused {eb:.2e} from complex128")
    assert ea <= max(1e-4, 3 * eb), (ea, eb)
    # complex64 CGLS drifts from complex128 after a few steps (loss of
    # orthogonality; fused and unfused alike): the early residuals agree
    for r, r3 in zip(rep, rep3):
        np.testing.assert_allclose(r.residual_history[:4], r3.residual_history[:4], rtol=1e-4)


@pytest.mark.parametrize("algo,kind", [("sirt", "hamming"), ("cgls", "none"), ("tv", "none")])
def test_graph_replay_matches_eager(sb, algo, kind):
    """Iterations 2.. replay a CUDA graph captured from iteration 1; the same
    solve issued eagerly (SPTB_NO_GRAPH) launches the same kernels in the
    same order: bitwise identical reconstructions and histories."""
    import torch
    from paper_2003_12677_b200.solvers import solve_batch
    ops = _ops(sb, 512, 96, kind)
    g = torch.Generator(device="cuda").manual_seed(5)
    sino = ops.radon(torch.rand(6, 512, 512, device="cuda", generator=g))
    cfg = sb.SolverConfig(algorithm=algo, max_iter=5)
    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    with _env("SPTB_NO_GRAPH", "1"):
        rec2, rep2, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    a = np.asarray(rec.cpu() if hasattr(rec, "cpu") else rec)
    b = np.asarray(rec2.cpu() if hasattr(rec2, "cpu") else rec2)
    np.testing.assert_array_equal(a, b)
    for r, r2 in zip(rep, rep2):
        assert r.residual_history == r2.residual_history
