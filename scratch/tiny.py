import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ops = sb.build_operators(sb.ScanGeometry(n_p=n, n_theta=45), filter_kind="ramlak")
u = torch.rand(4, n, n, device="cuda")
s = ops.radon(u); torch.cuda.synchronize(); print("ok", float(s.abs().sum()))
