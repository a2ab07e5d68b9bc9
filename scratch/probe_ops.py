import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
t=time.time()
geom = sb.ScanGeometry(n_p=2048, n_theta=1536)
ops = sb.build_operators(geom, filter_kind="ramlak", max_batch=32)
torch.cuda.synchronize(); print("build_operators c2: %.2f s calib %.6f nnz %d" % (time.time()-t, ops.calib_scale, ops.csr.nnz), flush=True)
sino = torch.randn(64, 1536, 2048, device="cuda")
u = torch.randn(64, 2048, 2048, device="cuda")
for name, fn, x in (("iradon", ops.iradon, sino), ("radon", ops.radon, u)):
    for _ in range(2): fn(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): y = fn(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/5
    print(f"{name} 64 slices: {ms:.2f} ms -> {64/ms*1e3:.0f} slices/s", flush=True)
