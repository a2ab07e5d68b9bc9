"""A/B of the S kernels at c2 (B=32): row-segment kernel vs the row-gather
kernel (SPTB_SPMM_ROWS=1): time through sptb_time_spmm, and compare gridrec
outputs of both paths on the same sinograms."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
n_p, T = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 1536)))
ops = sb.build_operators(sb.ScanGeometry(n_p=n_p, n_theta=T), filter_kind="ramlak", max_batch=32)
plan = ops.plan
g = torch.Generator(device="cuda").manual_seed(0)
sino = torch.randn(64, T, n_p, device="cuda", generator=g)
res = {}
for mode in ("pairs", "rows"):
    os.environ["SPTB_SPMM_ROWS"] = "1" if mode == "rows" else "0"
    _lib.lib.sptb_reload_switches()
    ms, uin = C.c_double(), C.c_int64()
    _lib.check(_lib.lib.sptb_time_spmm(plan.h, 2, 32, 30, C.byref(ms), C.byref(uin)))
    rows, cols, nnz = plan.matrix_info(_lib.MAT_S)
    byt = 12 * nnz + 4 * (rows + 1) + 8 * 32 * (uin.value + rows)
    rec = ops.iradon(sino)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.iradon(sino)
    e1.record(); torch.cuda.synchronize()
    res[mode] = rec
    print(f"{mode}: S {ms.value:.4f} ms {byt / ms.value / 1e6:.0f} GB/s; gridrec step {e0.elapsed_time(e1)/10:.3f} ms", flush=True)
for m in ("pairs",):
    print(f"rel diff {m} vs rows:", float((res[m] - res["rows"]).norm() / res["rows"].norm()))
