"""Per-iteration time of SIRT / CGLS / TV at config-1 size (256^2 x 180), one
pair and 64 slices: where launch overhead dominates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
geom = sb.ScanGeometry(n_p=256, n_theta=180)
for algo, filt in (("sirt", "hamming"), ("cgls", "none"), ("tv", "none")):
    ops = sb.build_operators(geom, filter_kind=filt, max_batch=32)
    for nz in (2, 64):
        sino = torch.randn(nz, 180, 256, device="cuda")
        t = {}
        for k in (2, 12, 2, 12):
            cfg = sb.SolverConfig(algorithm=algo, max_iter=k)
            torch.cuda.synchronize()
            l0 = _lib.lib.sptb_launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sb.solvers.solve_batch(sino, ops, cfg, raise_on_failure=False)
            e1.record()
            torch.cuda.synchronize()
            t[k] = (min(t.get(k, (1e9,))[0], e0.elapsed_time(e1)), _lib.lib.sptb_launch_count() - l0)
        per = (t[12][0] - t[2][0]) / 10
        launches = (t[12][1] - t[2][1]) / 10
        print(f"{algo} c1 {nz} slices: {1e3 * per:.1f} us/iteration, {launches:.1f} launches/iteration", flush=True)
