import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_geom(d):
    """Oracle geometry / kernel objects from a golden fixture."""
    from oracle import OGeom, OKernel
    g = OGeom(n_p=int(d["n_p"]), n_theta=int(d["n_theta"]), angles=d["angles"],
              n_x=int(d["n_x"]), n_y=int(d["n_y"]), center=float(d["center"]))
    k = OKernel(family=str(d["k_family"]), width=int(d["k_width"]),
                beta=float(d["k_beta"]), sigma=float(d["k_sigma"]))
    return g, k


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
