"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``sptomo`` read-only from /root/reference/pkg/src and writes
``tests/golden/*.npz``.  The fixtures travel with the repo; the reference does
not (it is absent on the GPU box).  Nothing here is imported by the product.
"""

from __future__ import annotations

import os
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# (name, ScanGeometry kwargs, KernelSpec kwargs)
GEOMS = [
    ("g32", dict(n_p=32, n_theta=20), {}),
    ("godd", dict(n_p=33, n_theta=17, center=15.7), {}),
    ("grect", dict(n_p=24, n_theta=11, n_x=28, n_y=20), {}),
    ("gw5", dict(n_p=32, n_theta=16), dict(width=5)),
    ("ggauss", dict(n_p=32, n_theta=16), dict(family="gauss")),
    ("gangles", dict(n_p=16, n_theta=5,
                     angles=np.array([0.3, 1.1, 2.0, 3.7, 5.9])), {}),
    ("c1", dict(n_p=256, n_theta=180), {}),
]

FILTERS = ("ramlak", "hamming", "shepplogan")


def _phantom_like(sp, geom):
    n = min(geom.n_x, geom.n_y)
    img = np.zeros(geom.grid_shape)
    ph = sp.phantom_shepp_logan(n)[0]
    img[:n, :n] = ph
    return img


def operators_case(sp, name, gkw, kkw):
    geom = sp.ScanGeometry(**gkw)
    kern = sp.KernelSpec(**kkw)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    ops = sp.build_operators(geom, kernel=kern, filter_kind="none")
    u = _phantom_like(sp, geom)
    lite = geom.n_grid > 20000  # config-1 size: phantom-derived inputs only
    if lite:
        # complex pair = (phantom, 0.5 * transposed phantom); sino = radon(u)
        uc = u + 0.5j * u.T
        s = ops.radon(u)
        sc = ops.radon(uc)
    else:
        uc = rng.standard_normal(geom.grid_shape) + 1j * rng.standard_normal(geom.grid_shape)
        s = rng.standard_normal(geom.sino_shape)
        sc = rng.standard_normal(geom.sino_shape) + 1j * rng.standard_normal(geom.sino_shape)
    out = dict(
        n_p=geom.n_p, n_theta=geom.n_theta, n_x=geom.n_x, n_y=geom.n_y,
        center=geom.center, angles=geom.angles,
        k_family=kern.family, k_width=kern.width, k_beta=kern.beta, k_sigma=kern.sigma,
        nnz=ops.csr.nnz, deapo=ops.deapo.values,
        u=u, uc=uc, s=s, sc=sc,
        radon_u=ops.radon(u), radon_uc=ops.radon(uc),
        adj_s=ops.radon_adjoint(s), adj_sc=ops.radon_adjoint(sc),
        S_row_ptr=ops.csr.row_ptr.astype(np.int64),
        SH_row_ptr=ops.csr.adj_row_ptr.astype(np.int64),
        S_abs_sum=float(np.abs(ops.csr.vals).sum()),
        S_val_sum=complex(ops.csr.vals.sum()),
    )
    small = geom.n_samples * 9 < 20000
    if small:
        out.update(S_col_idx=ops.csr.col_idx, S_vals=ops.csr.vals,
                   SH_col_idx=ops.csr.adj_col_idx, SH_vals=ops.csr.adj_vals)
    if lite:
        # drop fields the consumer can recompute bit-exactly
        for key in ("s", "sc", "uc"):
            out.pop(key)
        out["S_row_ptr"] = out["S_row_ptr"].astype(np.int32)
        out["SH_row_ptr"] = out["SH_row_ptr"].astype(np.int32)
    for kind in (FILTERS[:1] if lite else FILTERS):
        fops = sp.build_operators(geom, kernel=kern, filter_kind=kind)
        out[f"calib_{kind}"] = fops.calib_scale
        out[f"iradon_{kind}_radon_u"] = fops.iradon(out["radon_u"])
        if not lite:
            out[f"iradon_{kind}_s"] = fops.iradon(s)
            out[f"apply_{kind}_s"] = fops.apply_weights(s)
            out[f"apply_{kind}_sc"] = fops.apply_weights(sc)
    return out


def solvers_case(sp):
    """Paired / separate solver runs on the test_solvers.py:354-368 setup."""
    geom = sp.ScanGeometry(n_p=32, n_theta=20)
    yy, xx = np.mgrid[0:32, 0:32]
    a = np.clip(14 - np.hypot(xx - 16, yy - 16), 0, 1) * 0.8
    b = (np.hypot(xx - 12, yy - 18) < 6).astype(float)
    out = dict(slice_a=a, slice_b=b)
    rng = np.random.default_rng(5)
    for algo, iters in (("fbp", 1), ("sirt", 8), ("cgls", 8), ("tv", 5)):
        cfg = sp.SolverConfig(algorithm=algo, max_iter=iters)
        ops = sp.build_operators(geom, filter_kind=cfg.filter_kind())
        sa = ops.radon(a)
        sb = ops.radon(b) + 0.01 * rng.standard_normal(geom.sino_shape)
        out[f"{algo}_sino_a"] = sa
        out[f"{algo}_sino_b"] = sb
        rp, rep_p = sp.solve(sp.pair_complex(sa, sb), ops, cfg)
        ra, rep_a = sp.solve(sa, ops, cfg)
        out[f"{algo}_rec_pair"] = rp
        out[f"{algo}_rec_a"] = ra
        out[f"{algo}_hist_pair"] = np.asarray(rep_p.residual_history)
        out[f"{algo}_hist_a"] = np.asarray(rep_a.residual_history)
        out[f"{algo}_iters_pair"] = rep_p.iterations_run
        out[f"{algo}_conv_pair"] = rep_p.converged
    # nonneg / no-BB / tol variants
    ops_h = sp.build_operators(geom, filter_kind="hamming")
    sa = out["sirt_sino_a"]
    for tag, cfg in (("sirt_nobb", sp.SolverConfig(algorithm="sirt", max_iter=6, bb_enabled=False)),
                     ("sirt_nonneg", sp.SolverConfig(algorithm="sirt", max_iter=6, nonneg=True)),
                     ("sirt_tol", sp.SolverConfig(algorithm="sirt", max_iter=50, tol=0.05))):
        r, rep = sp.solve(sa, ops_h, cfg)
        out[f"{tag}_rec"] = r
        out[f"{tag}_hist"] = np.asarray(rep.residual_history)
        out[f"{tag}_iters"] = rep.iterations_run
    ops_n = sp.build_operators(geom, filter_kind="none")
    cfg = sp.SolverConfig(algorithm="tv", max_iter=3, mu=0.5, filter="none")
    r, rep = sp.solve(out["tv_sino_a"], ops_n, cfg)
    out["tv_mu_rec"] = r
    out["tv_mu_hist"] = np.asarray(rep.residual_history)
    return out


def cgs_case(sp):
    """cgs_mode=True runs of solve_cgls (solvers.py:247-248,262-305) on the
    solvers_case setup: paired and single, filter none and hamming, nonneg, tol."""
    geom = sp.ScanGeometry(n_p=32, n_theta=20)
    yy, xx = np.mgrid[0:32, 0:32]
    a = np.clip(14 - np.hypot(xx - 16, yy - 16), 0, 1) * 0.8
    b = (np.hypot(xx - 12, yy - 18) < 6).astype(float)
    rng = np.random.default_rng(7)
    out = {}
    for kind in ("none", "hamming"):
        ops = sp.build_operators(geom, filter_kind=kind)
        sa = ops.radon(a)
        sb = ops.radon(b) + 0.01 * rng.standard_normal(geom.sino_shape)
        out[f"{kind}_sino_a"] = sa
        out[f"{kind}_sino_b"] = sb
        for tag, cfg in (("", sp.SolverConfig(algorithm="cgls", max_iter=8, cgs_mode=True, filter=kind)),
                         ("_nonneg", sp.SolverConfig(algorithm="cgls", max_iter=6, cgs_mode=True,
                                                     nonneg=True, filter=kind)),
                         ("_tol", sp.SolverConfig(algorithm="cgls", max_iter=40, cgs_mode=True,
                                                  tol=0.02, filter=kind))):
            rp, rep_p = sp.solve(sp.pair_complex(sa, sb), ops, cfg)
            ra, rep_a = sp.solve(sa, ops, cfg)
            out[f"{kind}{tag}_rec_pair"] = rp
            out[f"{kind}{tag}_rec_a"] = ra
            out[f"{kind}{tag}_hist_pair"] = np.asarray(rep_p.residual_history)
            out[f"{kind}{tag}_hist_a"] = np.asarray(rep_a.residual_history)
            out[f"{kind}{tag}_conv_pair"] = rep_p.converged
            out[f"{kind}{tag}_conv_a"] = rep_a.converged
    return out


def precondition_case(sp):
    """precondition_apply / TomoOperators.precondition / preconditioner
    (operators.py:85-121,262-290): radial and per-sample weights, real and
    complex sinograms, a sinogram of another angle count, one detector row."""
    geom = sp.ScanGeometry(n_p=32, n_theta=20)
    rng = np.random.default_rng(9)
    s = rng.standard_normal(geom.sino_shape)
    sc = s + 1j * rng.standard_normal(geom.sino_shape)
    out = dict(s=s, sc=sc)
    for kind in ("hamming", "ramlak", "none"):
        ops = sp.build_operators(geom, filter_kind="ramlak")
        pre = ops.preconditioner(kind)
        out[f"pre_{kind}_w"] = pre.weights
        out[f"pre_{kind}_s"] = sp.precondition_apply(pre, s)
        out[f"pre_{kind}_sc"] = sp.precondition_apply(pre, sc)
    ops_h = sp.build_operators(geom, filter_kind="hamming")
    out["ops_hamming_precondition_s"] = ops_h.precondition(s)
    wfull = rng.uniform(0.0, 2.0, geom.sino_shape)
    pre = sp.Preconditioner(weights=wfull)
    out["wfull"] = wfull
    out["pre_full_sc"] = sp.precondition_apply(pre, sc)
    s7 = rng.standard_normal((7, 32))
    out["s7"] = s7
    out["pre_hamming_s7"] = sp.precondition_apply(ops.preconditioner("hamming"), s7)
    out["pre_hamming_row"] = sp.precondition_apply(ops.preconditioner("hamming"), s7[3])
    return out


def threshold_case(sp):
    """build_operators(..., threshold=0.05) (operators.py:317-371,
    gridding.py:159-195): both matrices pruned, the filtered one on its
    weighted values; operators and calibration on the pruned matrices."""
    geom = sp.ScanGeometry(n_p=32, n_theta=20)
    ops = sp.build_operators(geom, filter_kind="ramlak", threshold=0.05)
    rng = np.random.default_rng(11)
    u = rng.standard_normal(geom.grid_shape)
    s = rng.standard_normal(geom.sino_shape)
    out = dict(u=u, s=s, calib=ops.calib_scale, radon_u=ops.radon(u), iradon_s=ops.iradon(s),
               adj_s=ops.radon_adjoint(s))
    for tag, m in (("S", ops.csr), ("SF", ops.csr_filtered)):
        out[f"{tag}_row_ptr"] = m.row_ptr
        out[f"{tag}_col"] = m.col_idx
        out[f"{tag}_vals"] = m.vals
    return out


def cli_case(sp):
    """The reference CLI end to end (cli.py:111-161): phantom sinogram volume
    (odd slice count, noise) -> recon fbp / sirt-4 / cgls-3 (+ metrics JSON)
    and an intensity volume of the same stack -> recon fbp."""
    import json
    import tempfile
    from sptomo.cli import main as cli
    out = {}
    with tempfile.TemporaryDirectory() as td:
        sino = os.path.join(td, "sino.spt")
        assert cli(["phantom", "--size", "32", "--slices", "3", "--angles", "20", "--noise", "0.01",
                    "--seed", "4", "--out", sino]) == 0
        out["sino_bytes"] = np.frombuffer(open(sino, "rb").read(), dtype=np.uint8)
        for algo, iters in (("fbp", 1), ("sirt", 4), ("cgls", 3)):
            rec = os.path.join(td, f"rec_{algo}.spt")
            met = os.path.join(td, f"met_{algo}.json")
            assert cli(["recon", "--in", sino, "--out", rec, "--algo", algo, "--iters", str(iters),
                        "--metrics-out", met]) == 0
            out[f"rec_{algo}"] = sp.read_volume(rec).data
            out[f"hist_{algo}"] = np.asarray(json.load(open(met))[0]["residual_history"])
        v = sp.read_volume(sino)
        inten = os.path.join(td, "int.spt")
        sp.write_volume(inten, sp.io.KIND_INTENSITY, sp.io.simulate_intensity(v.data, 1.0),
                        center=v.center, angles=v.angles)
        out["int_bytes"] = np.frombuffer(open(inten, "rb").read(), dtype=np.uint8)
        rec = os.path.join(td, "rec_int.spt")
        assert cli(["recon", "--in", inten, "--out", rec, "--algo", "fbp"]) == 0
        out["rec_int_fbp"] = sp.read_volume(rec).data
    return out


def pipeline_case(sp):
    """run_pipeline on an odd 5-slice stack (test_pipeline.py:131-136)."""
    geom = sp.ScanGeometry(n_p=32, n_theta=12, n_z=5)
    ops = sp.build_operators(geom, filter_kind="ramlak")
    yy, xx = np.mgrid[0:32, 0:32]
    data = np.stack([ops.radon(np.clip(12 - np.hypot(xx - 16, yy - 16), 0, 1) * (1.0 - 0.05 * k))
                     for k in range(5)])
    stack = sp.SinogramStack(data=data, geometry=geom)
    out = {"stack": data}
    for algo, iters in (("fbp", 1), ("sirt", 4)):
        cfg = sp.SolverConfig(algorithm=algo, max_iter=iters)
        o = sp.build_operators(geom, filter_kind=cfg.filter_kind())
        vol, rep = sp.run_pipeline(stack, cfg, ops=o)
        out[f"{algo}_vol"] = vol.data
        out[f"{algo}_res"] = np.asarray(rep.residual_history)
        out[f"{algo}_iters"] = rep.iterations_run
    return out


DENSITY_GEOMS = ("g32", "godd", "c1")


def density_case(sp, name, gkw, kkw):
    """density_filter_solve (operators.py:189-236) and the density-filtered
    operators built on it (build_operators(filter_kind="density"))."""
    geom = sp.ScanGeometry(**gkw)
    kern = sp.KernelSpec(**kkw)
    ops = sp.build_operators(geom, kernel=kern, filter_kind="density")
    fs = ops.filter_spec
    sino = ops.radon(_phantom_like(sp, geom))
    return dict(n_p=geom.n_p, n_theta=geom.n_theta, weights=fs.weights,
                residual_history=np.asarray(fs.residual_history), converged=fs.converged,
                final_residual=fs.final_residual, calib=ops.calib_scale, sino=sino,
                iradon=ops.iradon(sino), **_geom_fields(geom, kern))


def _geom_fields(geom, kern):
    return dict(angles=geom.angles, n_x=geom.n_x, n_y=geom.n_y, center=geom.center,
                k_family=kern.family, k_width=kern.width, k_beta=kern.beta, k_sigma=kern.sigma)


def main():
    sys.path.insert(0, REF)
    import sptomo as sp  # noqa: E402  (the unmodified reference)
    for name, gkw, kkw in GEOMS:
        if name in DENSITY_GEOMS:
            np.savez_compressed(os.path.join(OUT, f"density_{name}.npz"), **density_case(sp, name, gkw, kkw))
            print("wrote density", name)
    if "--density-only" in sys.argv:
        return
    np.savez_compressed(os.path.join(OUT, "solvers_cgs_g32.npz"), **cgs_case(sp))
    print("wrote cgs")
    if "--cgs-only" in sys.argv:
        return
    np.savez_compressed(os.path.join(OUT, "precond_g32.npz"), **precondition_case(sp))
    print("wrote precond")
    if "--precond-only" in sys.argv:
        return
    np.savez_compressed(os.path.join(OUT, "threshold_g32.npz"), **threshold_case(sp))
    print("wrote threshold")
    if "--threshold-only" in sys.argv:
        return
    np.savez_compressed(os.path.join(OUT, "cli_g32.npz"), **cli_case(sp))
    print("wrote cli")
    if "--cli-only" in sys.argv:
        return
    for name, gkw, kkw in GEOMS:
        d = operators_case(sp, name, gkw, kkw)
        np.savez_compressed(os.path.join(OUT, f"ops_{name}.npz"), **d)
        print("wrote", name, "nnz", d["nnz"])
    np.savez_compressed(os.path.join(OUT, "solvers_g32.npz"), **solvers_case(sp))
    np.savez_compressed(os.path.join(OUT, "pipeline_g32.npz"), **pipeline_case(sp))
    print("done")


if __name__ == "__main__":
    main()


def cache_keys(sp):
    """Digests of make_cache_key (gridding.py:209-217) -> cache_keys.json
    (written by the one-off snippet in the round-1 history; kept here for
    regeneration)."""
    import json
    cases = [dict(n_p=32, n_theta=20), dict(n_p=33, n_theta=17, center=15.7),
             dict(n_p=24, n_theta=11, n_x=28, n_y=20), dict(n_p=256, n_theta=180)]
    out = []
    for gkw in cases:
        for kkw in ({}, dict(width=5), dict(family="gauss")):
            g, k = sp.ScanGeometry(**gkw), sp.KernelSpec(**kkw)
            for f in ("none", "ramlak", "density"):
                out.append(dict(geom=gkw, kernel=kkw, filter=f, digest=sp.make_cache_key(g, k, f).digest))
    with open(os.path.join(OUT, "cache_keys.json"), "w") as fh:
        json.dump(out, fh, indent=0)
