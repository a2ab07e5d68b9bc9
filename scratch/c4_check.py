"""BASELINE configs[3] geometry (2560^2 x 2048 angles): build, operator
identities and a short CGLS on the device (parity at full size is checked by
properties; the oracle is too slow here)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_12677_b200 as sb
torch.cuda.set_device(0)
g = sb.ScanGeometry(n_p=2560, n_theta=2048)
t = time.time(); ops = sb.build_operators(g, filter_kind="none", max_batch=32); torch.cuda.synchronize()
print("build %.2f s nnz %d" % (time.time() - t, ops.csr.nnz), flush=True)
gen = torch.Generator(device="cuda").manual_seed(0)
u = torch.randn(8, 2560, 2560, device="cuda", generator=gen)
s = torch.randn(8, 2048, 2560, device="cuda", generator=gen)
Ru, Rts = ops.radon(u), ops.radon_adjoint(s)
lhs = float((Ru.double() * s.double()).sum()); rhs = float((u.double() * Rts.double()).sum())
print("adjoint identity rel", abs(lhs - rhs) / abs(lhs), flush=True)
lin = ops.radon(u[:2] * 2.0 + u[2:4]) - (2 * Ru[:2] + Ru[2:4])
print("linearity rel", float(lin.norm() / Ru[:2].norm()), flush=True)
for name, fn, x in (("radon", ops.radon, torch.randn(64, 2560, 2560, device="cuda")), ("adjoint", ops.radon_adjoint, torch.randn(64, 2048, 2560, device="cuda"))):
    fn(x); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(x); e1.record(); torch.cuda.synchronize()
    print(f"{name} 64 slices: {e0.elapsed_time(e1):.2f} ms", flush=True)
cfg = sb.SolverConfig(algorithm="cgls", max_iter=5)
sino = ops.radon(u[:4])
t = time.time(); out, reps, st = sb.solvers.solve_batch(sino, ops, cfg, raise_on_failure=False); torch.cuda.synchronize()
print("cgls-5 %.2f s, iters %s, final res %s" % (time.time() - t, [r.iterations_run for r in reps], [round(r.residual_history[-1], 3) for r in reps]), flush=True)
