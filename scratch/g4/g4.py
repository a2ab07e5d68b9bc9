"""Drive scratch/g4/g4.cu on the c2 S pattern (CSR order, row-major rows)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2003_12677_b200 as sb
from paper_2003_12677_b200 import _lib
torch.cuda.set_device(0)
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libg4.so"))
ops = sb.build_operators(sb.ScanGeometry(n_p=2048, n_theta=1536), filter_kind="none", max_batch=32)
rows, cols, nnz = ops.plan.matrix_info(_lib.MAT_S)
rp = np.empty(rows + 1, np.int32); ci = np.empty(nnz, np.int32); v = np.empty(2 * nnz)
_lib.check(_lib.lib.sptb_plan_matrix_copy(ops.plan.h, _lib.MAT_S, rp.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
# device rows are row-major already in the copy's row order? (matrix_copy returns row-major rows m)
n = (nnz // 64) * 64
idx = torch.tensor(ci[:n], dtype=torch.int32, device="cuda")
x = torch.randn(cols, 64, device="cuda")  # 256-byte rows
ms = C.c_float()
for mode, name in ((1, "ldg128 half-warp/row"), (2, "ldg32 warp/row 1 line/instr"), (3, "ldg64 warp/row 2 lines/instr")):
    for grid in (148 * 2, 148 * 4, 148 * 8):
        rc = lib.g4_run(C.c_void_p(x.data_ptr()), C.c_longlong(cols), C.c_void_p(idx.data_ptr()), C.c_longlong(n), mode, grid, C.byref(ms))
        print(f"{name} grid {grid}: rc {rc}  {ms.value:.3f} ms  {n * 256 / ms.value / 1e6:.0f} GB/s gathered", flush=True)
