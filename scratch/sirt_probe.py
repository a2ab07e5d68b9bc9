import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
geom = sb.ScanGeometry(n_p=2048, n_theta=1536)
ops = sb.build_operators(geom, filter_kind=os.environ.get("FILT", "hamming"), max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda")
ks = [int(x) for x in (sys.argv[1:] or ["1", "6", "1", "6", "1", "6"])]
for k in ks:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out, reps, st = sb.solvers.solve_batch(sino, ops, sb.SolverConfig(algorithm=os.environ.get("ALGO", "sirt"), max_iter=k), raise_on_failure=False)
    e1.record()
    torch.cuda.synchronize()
    print(k, round(e0.elapsed_time(e1), 2), "ms", "its", min(r.iterations_run for r in reps), flush=True)
