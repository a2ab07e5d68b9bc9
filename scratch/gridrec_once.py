"""Three gridrec launches at c2 (64 slices, B=32) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
ops = sb.build_operators(sb.ScanGeometry(n_p=2048, n_theta=1536), filter_kind="ramlak", max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda")
for _ in range(int(os.environ.get("REPS", "3"))):
    rec = ops.iradon(sino)
torch.cuda.synchronize()
print("ok", float(rec[0].abs().mean()))
