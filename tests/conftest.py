import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: minutes of host work; opt-in via DGM_SLOW=1")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_refelem():
    return load_golden("refelem.npz")


def golden_element(ref: dict, n: int):
    """Reference element assembled from the golden arrays (independent of the product)."""
    nodes = ref[f"n{n}_nodes"]
    return SimpleNamespace(
        order=n, num_nodes=len(nodes), num_face_nodes=ref[f"n{n}_face_nodes"].shape[1],
        nodes=nodes, diff=ref[f"n{n}_diff"], lift=ref[f"n{n}_lift"], mass=ref[f"n{n}_mass"],
        face_mass=ref[f"n{n}_face_mass"], face_barycentrics=ref[f"n{n}_face_barycentrics"],
        face_nodes=ref[f"n{n}_face_nodes"].astype(np.int64))


def rel_l2(got, want) -> float:
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want.ravel())
    return float(np.linalg.norm((got - want).ravel()) / (den if den > 0 else 1.0))


def rel_max(got, want) -> float:
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    scale = np.abs(want).max()
    return float(np.abs(got - want).max() / (scale if scale > 0 else 1.0))
