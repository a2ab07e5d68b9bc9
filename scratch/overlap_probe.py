"""Two gridrec batches (64 slices each, two plans) back to back on one stream
vs concurrently on two streams: does S (L2-bound) overlap the HBM-bound FFT
passes?  SPTB_PERSIST_SMS limits the persistent FFT kernels' CTAs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
g = sb.ScanGeometry(n_p=2048, n_theta=1536)
A = sb.build_operators(g, filter_kind="ramlak", max_batch=32)
Bo = sb.build_operators(g, filter_kind="ramlak", max_batch=32)
sino = torch.randn(64, 1536, 2048, device="cuda")
oa = torch.empty(64, 2048, 2048, device="cuda"); ob = torch.empty_like(oa)
sa, sbs = torch.cuda.Stream(), torch.cuda.Stream()
from paper_2003_12677_b200 import _lib
import ctypes as C
fmt = _lib.FMT_F32 | _lib.FMT_REAL
def run(ops, out):
    _lib.check(_lib.lib.sptb_iradon(ops.plan.h, C.c_void_p(sino.data_ptr()), fmt, C.c_void_p(out.data_ptr()), fmt, 64))
def timeit(f, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for _ in range(reps): f()
    ev = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    e1.record(torch.cuda.current_stream()); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
cur = torch.cuda.current_stream()
A.plan.bind_stream(cur.cuda_stream); Bo.plan.bind_stream(cur.cuda_stream)
for _ in range(3): run(A, oa); run(Bo, ob)
seq = min(timeit(lambda: (run(A, oa), run(Bo, ob))) for _ in range(3))
A.plan.bind_stream(sa.cuda_stream); Bo.plan.bind_stream(sbs.cuda_stream)
def conc_many(reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    sa.wait_stream(cur); sbs.wait_stream(cur)
    for _ in range(reps):
        run(A, oa); run(Bo, ob)
    cur.wait_stream(sa); cur.wait_stream(sbs)
    e1.record(cur); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
conc_many(3)
par = min(conc_many() for _ in range(3))
print(f"SMS={os.environ.get('SPTB_PERSIST_SMS','all')}: two batches sequential {seq:.3f} ms, concurrent {par:.3f} ms -> {par/2:.3f} ms per batch")
