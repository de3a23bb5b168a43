import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built native library")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def perturbed_mesh2():
    """2x2x2 mesh with perturbed geometry (reference tests/conftest.py:7-10)."""
    from paper_1711_00903_b200.mesh import build_cube_mesh, perturb_mesh
    return perturb_mesh(build_cube_mesh(2, 2.0), amplitude=0.15, seed=7)


@pytest.fixture(scope="session")
def perturbed_single():
    """One perturbed element (reference tests/conftest.py:13-16)."""
    from paper_1711_00903_b200.mesh import build_cube_mesh, perturb_mesh
    return perturb_mesh(build_cube_mesh(1, 2.0), amplitude=0.2, seed=11)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
