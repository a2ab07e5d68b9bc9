"""Parity at the headline configuration (BASELINE configs[1], north_star
"Target"): 2048^2 x 1536 angles, a 64-slice batch = 32 complex vectors per
launch, i.e. exactly the kernel instantiations bench.py times:

* gridrec: fused FFT1 column pass (radix-16, n_p = 2^11) -> S diag(w) row
  gather over the c2 matrix (DC row of 4,852 nonzeros: chunked long-row path)
  -> FFT2 y pass -> FFT2 x pass + deapodization + unpack;
* radon: FFT2 x pass + pack + deapodization -> y pass -> S^H (TMA slot
  kernel, sample-order rows) -> inverse FFT1 column pass;
* SIRT-5 (Hamming, BB) with the element passes fused into the FFT2 x passes.

Checked against the oracle (the reference algorithm, operators.py:153-187,
solvers.py:133-186, restated in oracle/ and pinned by tests/golden) on slices
{0, 1, 31, 62, 63}: north_star's 1e-4 relative L2 per operator application
and 1e-3 after the stated solver iterations.  Each slice of the batch is
distinct (scaled phantom + per-slice noise), so slot mix-ups would show.
"""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]

N_P, N_T, NZ = 2048, 1536, 64
CHECK = (0, 1, 31, 62, 63)
PAIRS = sorted({s // 2 for s in CHECK})


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2003_12677_b200 as sb
    from oracle import OGeom, build_oracle_ops, shepp_logan
    from oracle import parity
    og = OGeom(N_P, N_T)
    o_ram = build_oracle_ops(og, kind="ramlak")
    o_ham = build_oracle_ops(og, kind="hamming")
    parity.register("ramlak", o_ram)
    parity.register("hamming", o_ham)
    ph = shepp_logan(N_P, 2)
    base = o_ram.radon(ph[0] + 1j * ph[1])          # oracle sinogram pair of the phantom
    geom = sb.ScanGeometry(n_p=N_P, n_theta=N_T)
    return dict(sb=sb, torch=torch, parity=parity, ph=ph,
                base=np.stack([base.real, base.imag]), geom=geom)


def _stack(torch, two, noise, seed):
    """64 distinct slices: scale_z * two[z % 2] + noise * N(0,1) (float32, device)."""
    dev = torch.device("cuda")
    t = torch.tensor(two, dtype=torch.float32, device=dev)
    sc = torch.linspace(1.0, 0.8, NZ, device=dev)
    g = torch.Generator(device=dev).manual_seed(seed)
    x = t[torch.arange(NZ, device=dev) % 2] * sc[:, None, None]
    return (x + noise * torch.randn(x.shape, device=dev, generator=g)).contiguous()


def test_gridrec_headline_batch(env):
    sb, torch, parity = env["sb"], env["torch"], env["parity"]
    ops = sb.build_operators(env["geom"], filter_kind="ramlak", max_batch=32)
    amp = float(np.abs(env["base"]).max())
    sino = _stack(torch, env["base"], 0.01 * amp, seed=11)
    rec = ops.iradon(sino)
    torch.cuda.synchronize()
    sh = sino.cpu().numpy()
    rh = rec.cpu().numpy()
    want = parity.run([("iradon", "ramlak", parity.pair_of(sh, k), {}) for k in PAIRS])
    for k, w in zip(PAIRS, want):
        for z, part in ((2 * k, w.real), (2 * k + 1, w.imag)):
            if z in CHECK:
                e = parity.rel_l2(rh[z], part)
                assert e < 1e-4, (z, e)


def test_radon_headline_batch(env):
    sb, torch, parity = env["sb"], env["torch"], env["parity"]
    ops = sb.build_operators(env["geom"], filter_kind="ramlak", max_batch=32)
    img = _stack(torch, env["ph"], 0.02, seed=12)
    sino = ops.radon(img)
    torch.cuda.synchronize()
    ih = img.cpu().numpy()
    shh = sino.cpu().numpy()
    want = parity.run([("radon", "ramlak", parity.pair_of(ih, k), {}) for k in PAIRS])
    for k, w in zip(PAIRS, want):
        for z, part in ((2 * k, w.real), (2 * k + 1, w.imag)):
            if z in CHECK:
                e = parity.rel_l2(shh[z], part)
                assert e < 1e-4, (z, e)


def test_sirt5_headline_batch(env):
    """SIRT-5 (Hamming, BB, u0 = 0) on the 64-slice batch with 2% noise
    (BASELINE configs[2] data model) vs the oracle on pairs 0, 15, 31."""
    sb, torch, parity = env["sb"], env["torch"], env["parity"]
    ops = sb.build_operators(env["geom"], filter_kind="hamming", max_batch=32)
    amp = float(np.abs(env["base"]).max())
    sino = _stack(torch, env["base"], 0.02 * amp, seed=13)
    cfg = sb.SolverConfig(algorithm="sirt", max_iter=5)
    rec, reps, stat = sb.solvers.solve_batch(sino, ops, cfg)
    torch.cuda.synchronize()
    assert stat == [0] * (NZ // 2)
    sh = sino.cpu().numpy()
    rh = rec.cpu().numpy()
    want = parity.run([("solve", "hamming", parity.pair_of(sh, k),
                        {"algorithm": "sirt", "max_iter": 5}) for k in PAIRS])
    for k, (u, hist, its, _conv) in zip(PAIRS, want):
        assert reps[k].iterations_run == its == 5
        e = parity.rel_l2(rh[2 * k] + 1j * rh[2 * k + 1], u)
        assert e < 1e-3, (k, e)
        eh = parity.rel_l2(reps[k].residual_history, hist)
        assert eh < 1e-3, (k, eh)


def test_headline_batch_properties(env):
    """Size-independent properties on all 64 slices of the production batch
    (every slot, not only the oracle-checked ones): adjointness of the radon
    pair <s, A u> = <A^H s, u> per slice, linearity of A, and slot
    independence -- a pair's gridrec does not depend on its batch slot
    (the stack rolled by 6 pairs gives the same slices bit for bit: fixed
    per-unit reduction order), and slice 37 alone (other kernels: a
    one-unit launch) agrees to rounding."""
    sb, torch = env["sb"], env["torch"]
    ops = sb.build_operators(env["geom"], filter_kind="ramlak", max_batch=32)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(21)
    u = torch.rand(NZ, N_P, N_P, device=dev, generator=g)
    s = torch.randn(NZ, N_T, N_P, device=dev, generator=g)
    au = ops.radon(u)
    ahs = ops.radon_adjoint(s)
    lhs = (s.double() * au.double()).sum(dim=(1, 2))
    rhs = (ahs.double() * u.double()).sum(dim=(1, 2))
    # complex64 kernels; s has random signs, so <s, A u> ~ sqrt(N) |terms| and
    # its relative rounding is ~1e-5 (the complex128 build meets 1e-8:
    # test_gpu_operators.py::test_adjoint_identity_and_linearity)
    err = ((lhs - rhs).abs() / lhs.abs().clamp_min(1e-30)).max().item()
    assert err < 1e-4, err
    v = torch.rand(NZ, N_P, N_P, device=dev, generator=g)
    lin = ops.radon(0.75 * u - 1.5 * v)
    ref = 0.75 * au - 1.5 * ops.radon(v)
    assert ((lin - ref).norm() / ref.norm()).item() < 1e-6
    rec = ops.iradon(s)
    rolled = ops.iradon(torch.roll(s, 12, dims=0).contiguous())
    one = ops.iradon(s[37:38].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(torch.roll(rolled, -12, dims=0), rec)
    # a lone slice is packed with a zero partner and runs the one-unit
    # kernels: rounding only
    assert ((one[0] - rec[37]).norm() / rec[37].norm()).item() < 1e-5
