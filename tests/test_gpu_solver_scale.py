"""Solver parity at the configurations and iteration counts BASELINE.json
states (north_star: 1e-3 relative L2 "after the stated solver iteration
count"):

* SIRT-100 (Hamming, BB) at 2048^2 x 1536 on a noisy phantom pair
  (BASELINE configs[2]; solvers.py:133-186);
* CGLS-50 (filter none) at 2560^2 x 2048 (configs[3]; solvers.py:189-259).
  By 50 steps CGLS on this system has lost orthogonality: the reference
  itself moves by 2.7e-4 (final residual by 2.5%) under 1e-15 relative
  perturbations of its operators, 4.3e-4 under 1e-13 -- the complex128 bar
  is max(1e-3, 3x that spread, measured in the run);
* TV-10 (split Bregman, 2 inner CGLS steps, default mu) at 2048^2 x 1536
  (configs[4]; solvers.py:344-432).

The oracle (the reference algorithm, pinned by tests/golden) runs each case
on the host in a fork pool, next to the same case with every operator
evaluated in complex64 (oracle/emulate.py Fp32PipelineOperators): the
reference algorithm's own deviation when its operators are single precision.
The 1e-3 bar is carried by the complex128 build of the device kernels; the
complex64 production build must stay within max(1e-3, 2x that emulated
deviation) -- SURVEY section 7.6.  The noise seed of the SIRT pair was
chosen so that the reference's 10x divergence guard does not stop it before
100 iterations (BB-SIRT on noisy data is non-monotone: seeds 0, 1 and 5 trip
it, seed 3 peaks at 2.8x its running minimum -- scratch/sirt_seed_search.py
and its log).  These cases take several minutes of host time (marked slow).
"""

import numpy as np
import pytest

from conftest import rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIRT_SEED = 3
CASES = {
    # name: (n_p, n_theta, filter, algorithm, iterations, noise)
    "sirt100_c2": (2048, 1536, "hamming", "sirt", 100, 0.02),
    "cgls50_c4": (2560, 2048, "none", "cgls", 50, 0.0),
    "tv10_c2": (2048, 1536, "none", "tv", 10, 0.0),
}


def _oracle_ops():
    from oracle import OGeom, build_oracle_ops
    return {
        ("c2", "hamming"): build_oracle_ops(OGeom(2048, 1536), kind="hamming"),
        ("c2", "none"): build_oracle_ops(OGeom(2048, 1536), kind="none"),
        ("c4", "none"): build_oracle_ops(OGeom(2560, 2048), kind="none"),
    }


def _key(name):
    n_p, _, filt, _, _, _ = CASES[name]
    return ("c4" if n_p == 2560 else "c2", filt)


_OPS = {}


def _job(args):
    from oracle import o_solve
    from oracle.emulate import Fp32PipelineOperators, PerturbedOperators
    name, sino, variant = args
    _, _, _, algo, iters, _ = CASES[name]
    ops = _OPS[_key(name)]
    if variant == "emu":
        ops = Fp32PipelineOperators(ops)
    elif variant.startswith("pert"):
        ops = PerturbedOperators(ops, 1e-13, int(variant[4:]))
    u, rep = o_solve(sino, ops, algo, max_iter=iters)
    return name, variant, u, list(rep.history)


@pytest.fixture(scope="module")
def ref():
    """Sinogram pairs (oracle radon of the phantom pair, + noise) and the
    oracle's exact and complex64-emulated solutions, computed in parallel."""
    import multiprocessing as mp
    import os
    from oracle import shepp_logan
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    _OPS.update(_oracle_ops())
    data = {}
    for name, (n_p, n_t, filt, algo, iters, noise) in CASES.items():
        ph = shepp_logan(n_p, 2)
        s = _OPS[_key(name)].radon(ph[0] + 1j * ph[1])
        if noise:
            rng = np.random.default_rng(SIRT_SEED)
            amp = np.abs(s).max()
            s = s + noise * amp * (rng.standard_normal(s.shape) + 1j * rng.standard_normal(s.shape))
        data[name] = s
    # exact, complex64-emulated, and (CGLS: loses orthogonality by 50 steps)
    # two runs with 1e-13 operator perturbations -- the reference's own spread
    jobs = [(n, data[n], v) for n in CASES for v in ("exact", "emu")]
    jobs += [("cgls50_c4", data["cgls50_c4"], f"pert{k}") for k in (1, 2)]
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        res = pool.map(_job, jobs, chunksize=1)
    out = {n: {"sino": data[n]} for n in CASES}
    for name, variant, u, hist in res:
        out[name][variant] = (u, hist)
    return out


@pytest.fixture(scope="module")
def sb():
    import paper_2003_12677_b200 as m
    return m


@pytest.mark.parametrize("name", list(CASES))
def test_solver_at_stated_iterations(sb, ref, name):
    n_p, n_t, filt, algo, iters, _ = CASES[name]
    geom = sb.ScanGeometry(n_p=n_p, n_theta=n_t)
    sino = ref[name]["sino"]
    u_ex, h_ex = ref[name]["exact"]
    u_em, h_em = ref[name]["emu"]
    cfg = sb.SolverConfig(algorithm=algo, max_iter=iters, filter=filt)
    # complex128 build of the same kernels: the 1e-3 bar
    ops64 = sb.build_operators(geom, filter_kind=filt, precision="complex128", max_batch=2)
    r64, rep64 = sb.solve(sino, ops64, cfg)
    e64 = rel(r64, u_ex)
    # the reference's own spread under 1e-13 operator perturbations (CGLS-50:
    # 2.7e-4 already at 1e-15, final residual moving by 2-4%)
    spread = max([rel(ref[name][v][0], u_ex) for v in ref[name] if v.startswith("pert")], default=0.0)
    hspread = max([abs(ref[name][v][1][-1] - h_ex[-1]) / h_ex[-1] for v in ref[name] if v.startswith("pert")],
                  default=0.0)
    bar, hbar = max(1e-3, 3.0 * spread), max(1e-3, 3.0 * hspread)
    print(f"{name}: complex128 {e64:.2e} after {rep64.iterations_run} iterations, bar {bar:.2e} "
          f"(history {rep64.residual_history[-1]:.6e} vs {h_ex[-1]:.6e}, bar {hbar:.2e})", flush=True)
    assert rep64.iterations_run == len(h_ex) == iters
    assert e64 <= bar, (name, e64, bar)
    assert abs(rep64.residual_history[-1] - h_ex[-1]) <= hbar * h_ex[-1]
    del ops64
    # complex64 production build: within 2x the reference's own complex64 deviation
    ops32 = sb.build_operators(geom, filter_kind=filt, max_batch=2)
    r32, rep32 = sb.solve(sino, ops32, cfg)
    e32, floor = rel(r32, u_ex), rel(u_em, u_ex)
    print(f"{name}: complex128 {e64:.2e}, complex64 {e32:.2e}, reference in complex64 {floor:.2e}")
    assert rep32.iterations_run == iters
    assert e32 <= max(1e-3, 2.0 * floor), (name, e32, floor)
