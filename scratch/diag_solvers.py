import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12677_b200 as sb
from oracle import OGeom, build_oracle_ops, o_solve, shepp_logan
sol = dict(np.load('tests/golden/solvers_g32.npz'))
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for prec in ("complex128", "complex64"):
    ops = sb.build_operators(sb.ScanGeometry(32, 20), filter_kind="none", precision=prec)
    for it in (1, 2, 3, 5):
        r, rep = sb.solve(sol["tv_sino_a"], ops, sb.SolverConfig(algorithm="tv", max_iter=it, mu=0.5))
        o = build_oracle_ops(OGeom(32, 20), kind="none")
        ro, orep = o_solve(sol["tv_sino_a"], o, "tv", max_iter=it, mu=0.5)
        print(prec, "tv it", it, rel(r, ro), rep.residual_history, orep.history)
    for it in (1, 2):
        r, rep = sb.solve(sol["tv_sino_a"], ops, sb.SolverConfig(algorithm="tv", max_iter=1, tv_inner_iter=it, mu=0.5))
        ro, orep = o_solve(sol["tv_sino_a"], o, "tv", max_iter=1, inner=it, mu=0.5)
        print(prec, "tv inner", it, rel(r, ro))
for prec in ("complex128", "complex64"):
    geom = sb.ScanGeometry(n_p=256, n_theta=180)
    ops = sb.build_operators(geom, filter_kind="none", precision=prec)
    oops = build_oracle_ops(OGeom(256, 180), kind="none")
    u = shepp_logan(256)[0]
    sino = oops.radon(u)
    for it in (1, 3, 10):
        r, rep = sb.solve(sino, ops, sb.SolverConfig(algorithm="cgls", max_iter=it))
        ro, orep = o_solve(sino, oops, "cgls", max_iter=it)
        print(prec, "cgls c1 it", it, rel(r, ro))
    # operator accuracy at c1
    print(prec, "radon err", rel(ops.radon(u), oops.radon(u)), "adj err", rel(ops.radon_adjoint(sino), oops.radon_adjoint(sino)))
