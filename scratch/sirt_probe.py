import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
geom = sb.ScanGeometry(n_p=2048, n_theta=1536)
ops = sb.build_operators(geom, filter_kind="hamming", max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda")
for k in (1, 3):
    out, reps, st = sb.solvers.solve_batch(sino, ops, sb.SolverConfig(algorithm="sirt", max_iter=k), raise_on_failure=False)
torch.cuda.synchronize()
print("ok")
