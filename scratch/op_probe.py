"""Time radon / iradon at c2 (64 slices, device tensors) and print kernel mix."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
ops = sb.build_operators(sb.ScanGeometry(n_p=2048, n_theta=1536), filter_kind="ramlak", max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda"); u = torch.randn(64, 2048, 2048, device="cuda")
for name, fn, x in (("iradon", ops.iradon, sino), ("radon", ops.radon, u)):
    for _ in range(2): fn(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): fn(x)
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1)/5:.3f} ms / 64 slices", flush=True)
