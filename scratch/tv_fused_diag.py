"""Fused vs unfused TV passes vs the complex128 build, per test case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
from paper_2003_12677_b200.solvers import solve_batch

def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))

def run(ops, sino, cfg, unfused):
    if unfused: os.environ["SPTB_XPASS_UNFUSED"] = "1"
    else: os.environ.pop("SPTB_XPASS_UNFUSED", None)
    _lib.lib.sptb_reload_switches()
    rec, rep, _ = solve_batch(sino, ops, cfg, raise_on_failure=False)
    rec = rec.cpu().numpy() if hasattr(rec, "cpu") else np.asarray(rec)
    return rec.astype(np.float64), rep

for (n, T, nx, ny, inner, nonneg) in [(512, 96, None, None, 2, False), (512, 96, None, None, 3, True),
                                      (512, 96, None, None, 1, False), (4096, 6, None, None, 2, False),
                                      (1024, 24, 512, 2048, 2, True), (512, 45, 1024, 512, 2, False)]:
    geom = sb.ScanGeometry(n_p=n, n_theta=T, n_x=nx, n_y=ny)
    ops = sb.build_operators(geom, filter_kind="none", max_batch=4)
    g = torch.Generator(device="cuda").manual_seed(n + T + inner)
    img = torch.rand(8, ops.geom.n_y, ops.geom.n_x, device="cuda", generator=g)
    sino = ops.radon(img)
    cfg = sb.SolverConfig(algorithm="tv", max_iter=4, tv_inner_iter=inner, nonneg=nonneg)
    a, ra = run(ops, sino, cfg, False)
    b, rb = run(ops, sino, cfg, True)
    ops64 = sb.build_operators(geom, filter_kind="none", max_batch=4, precision="complex128")
    c, rc = run(ops64, sino.double().cpu().numpy(), cfg, False)
    print((n, T, nx, ny, inner, nonneg), "fused-unfused %.2e fused-c128 %.2e unfused-c128 %.2e" % (rel(a, b), rel(a, c), rel(b, c)),
          [r.iterations_run for r in ra], [r.iterations_run for r in rb], [getattr(r, "status", None) for r in ra][:4],
          flush=True)
    print("   hist f", ra[0].residual_history, "\n   hist u", rb[0].residual_history, "\n   hist c", rc[0].residual_history, flush=True)
