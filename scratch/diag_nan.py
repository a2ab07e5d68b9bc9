import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_12677_b200 as sb
from oracle import shepp_logan
geom = sb.ScanGeometry(n_p=32, n_theta=12, n_z=8)
ops = sb.build_operators(geom, filter_kind="none")
data = np.stack([ops.radon(shepp_logan(32)[0] * (1 - 0.05 * k)) for k in range(8)])
data[0, 0, 0] = np.nan
for algo in ("tv", "sirt", "cgls", "fbp"):
    rec, reps, stat = sb.solvers.solve_batch(data, ops, sb.SolverConfig(algorithm=algo, max_iter=2, filter="none"), raise_on_failure=False)
    print(algo, stat, [r.iterations_run for r in reps], [r.converged for r in reps], np.isnan(rec).sum(), reps[0].residual_history)
