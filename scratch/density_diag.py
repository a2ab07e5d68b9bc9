import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, paper_2003_12677_b200 as sb
from conftest import load_golden, rel
from oracle import density_weights, build_gridding, OGeom, OKernel
for f in ("density_g32.npz", "density_c1.npz"):
    d = load_golden(f)
    g = sb.ScanGeometry(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]))
    for prec in ("complex128", "complex64"):
        ops = sb.build_operators(g, filter_kind="density", precision=prec)
        fs = ops.filter_spec
        h, hr = fs.residual_history, d["residual_history"]
        print(f, prec, "w rel", rel(fs.weights, d["weights"]), "hist n", len(h), len(hr),
              "hist rel first/last", abs(h[1]-hr[1])/hr[1], abs(h[-1]-hr[-1])/hr[-1], "final", fs.final_residual, float(d["final_residual"]))
    # oracle with float32-rounded magnitudes
    og = OGeom(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]))
    gr = build_gridding(og, OKernel())
    w, hh, c, fin = density_weights(gr, og)
    print("oracle rel", rel(w, d["weights"]))
from oracle import build_oracle_ops
d = load_golden("density_c1.npz")
og = OGeom(n_p=256, n_theta=180)
oo = build_oracle_ops(og, OKernel(), "density")
print("oracle calib on this box", oo.calib, "golden", float(d["calib"]), "iradon rel", rel(oo.iradon(d["sino"]), d["iradon"]))
