"""Time the production SpMM launches at c2 (B=32) through sptb_time_spmm."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
n_p, T = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 1536)))
reps = int(os.environ.get("REPS", "20"))
ops = sb.build_operators(sb.ScanGeometry(n_p=n_p, n_theta=T), filter_kind="ramlak", max_batch=32)
plan = ops.plan
for name, which in (("S_H", 1), ("S_filtered", 2)):
    ms, uin = C.c_double(), C.c_int64()
    _lib.check(_lib.lib.sptb_time_spmm(plan.h, which, 32, reps, C.byref(ms), C.byref(uin)))
    nnz = ops.csr.nnz
    rows = ops.geom.n_theta * ops.geom.n_p if which == 1 else ops.geom.n_p ** 2
    byt = 12 * nnz + 4 * (rows + 1) + 8 * 32 * (uin.value + rows)
    print(f"{name}: {ms.value:.4f} ms  {byt / ms.value / 1e6:.0f} GB/s  ({byt/1e9:.3f} GB model)", flush=True)
