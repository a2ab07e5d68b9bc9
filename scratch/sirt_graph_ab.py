"""SIRT / CGLS / TV per-iteration time at c2 (64 slices) with and without the
iteration graphs (SPTB_NO_GRAPH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
geom = sb.ScanGeometry(n_p=2048, n_theta=1536)
sino = torch.randn(64, 1536, 2048, device="cuda")
for algo, filt in (("sirt", "hamming"), ("cgls", "none")):
    ops = sb.build_operators(geom, filter_kind=filt, max_batch=32)
    for ng in ("0", "1"):
        os.environ["SPTB_NO_GRAPH"] = ng
        _lib.lib.sptb_reload_switches()
        t = {}
        for k in (2, 12, 2, 12):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sb.solvers.solve_batch(sino, ops, sb.SolverConfig(algorithm=algo, max_iter=k), raise_on_failure=False)
            e1.record()
            torch.cuda.synchronize()
            t[k] = min(t.get(k, 1e9), e0.elapsed_time(e1))
        print(f"{algo} no_graph={ng}: {(t[12] - t[2]) / 10:.3f} ms/iteration", flush=True)
