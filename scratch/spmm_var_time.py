"""Time the in-path S kernel (sptb_time_spmm, S diag(w), c2, B=32) of the
library variant named by SPTB_LIB_VARIANT (scratch/build_variant.sh)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
ops = sb.build_operators(sb.ScanGeometry(n_p=2048, n_theta=1536), filter_kind="ramlak", max_batch=32)
plan = ops.plan
rows, cols, nnz = plan.matrix_info(_lib.MAT_S)
for which in (2, 1):
    best = 1e9
    for _ in range(3):
        ms, uin = C.c_double(), C.c_int64()
        _lib.check(_lib.lib.sptb_time_spmm(plan.h, which, 32, 30, C.byref(ms), C.byref(uin)))
        best = min(best, ms.value)
    byt = 12 * nnz + 4 * (rows + 1) + 8 * 32 * (uin.value + rows)
    print(f"{os.environ.get('SPTB_LIB_VARIANT','libsptb.so')} which={which}: {best:.4f} ms {byt/best/1e6:.0f} GB/s", flush=True)
