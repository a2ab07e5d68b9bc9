import numpy as np, multiprocessing as mp, time, sys
from oracle import OGeom, build_oracle_ops, shepp_logan
from oracle.solvers import o_sirt, ODivergence
g = OGeom(2048, 1536)
t=time.time()
ops = build_oracle_ops(g, kind="hamming")
ph = shepp_logan(2048, 2)
base = ops.radon(ph[0] + 1j*ph[1])
print("setup", time.time()-t, flush=True)
def run(seed):
    rng = np.random.default_rng(seed)
    amp = np.abs(base).max()
    s = base + 0.02*amp*(rng.standard_normal(base.shape) + 1j*rng.standard_normal(base.shape))
    try:
        u, rep = o_sirt(s, ops, 100)
        h = np.array(rep.history); ratio = max(h[i]/h[:i+1].min() for i in range(len(h)))
        return seed, "ok", rep.iterations, ratio
    except ODivergence as e:
        return seed, "div", str(e)[:60], None
with mp.get_context("fork").Pool(8) as p:
    for r in p.imap_unordered(run, range(8)): print(r, time.time()-t, flush=True)
