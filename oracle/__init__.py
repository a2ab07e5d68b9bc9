"""CPU oracle for the sptomo hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain NumPy/SciPy restatement of the reference algorithm
(``/root/reference/pkg/src/sptomo``: geometry.py, gridding.py, operators.py,
solvers.py, pipeline.py).  Every function cites the reference file:line it
follows.  It exists to check the CUDA product path, never to be it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2003_12677_b200`` never imports it and has no
  CPU fallback.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by the unmodified reference package
(``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` exists; the fixtures travel, the reference does not).
"""

from .tomo import (OGeom, OKernel, build_gridding, deapodization, density_weights, filter_weights,
                   op_radon, op_radon_adjoint, op_iradon, op_apply_weights,
                   calibration_scale, OracleOps, build_oracle_ops,
                   shepp_logan, snr_db)
from .solvers import (o_solve, o_fbp, o_sirt, o_cgls, o_tv, OReport,
                      ODivergence, ONonFinite)

__all__ = [
    "OGeom", "OKernel", "build_gridding", "deapodization", "filter_weights",
    "op_radon", "op_radon_adjoint", "op_iradon", "op_apply_weights",
    "calibration_scale", "OracleOps", "build_oracle_ops", "shepp_logan",
    "snr_db", "o_solve", "o_fbp", "o_sirt", "o_cgls", "o_tv", "OReport",
    "ODivergence", "ONonFinite",
]
