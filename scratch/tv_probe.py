"""Launch mix of a short TV solve at 2048^2 x 1536 (64 slices): for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2003_12677_b200 as sb
from paper_2003_12677_b200.solvers import solve_batch
torch.cuda.set_device(0)
ops = sb.build_operators(sb.ScanGeometry(n_p=2048, n_theta=1536), filter_kind="none", max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda")
solve_batch(sino, ops, sb.SolverConfig(algorithm="tv", max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 2),
            raise_on_failure=False)
torch.cuda.synchronize()
