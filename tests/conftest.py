import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and the built libsisdc_b200.so")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return {name: np.load(os.path.join(GOLDEN, name + ".npz")) for name in ("tables", "operators", "trajectories", "nonincremental", "dirichlet", "presmooth", "htransfer", "cns", "sources", "study", "sod")}


@pytest.fixture(scope="session")
def golden_ml():
    import numpy as np
    return np.load(os.path.join(GOLDEN, "multilevel.npz"))


@pytest.fixture(scope="session")
def golden_mls():
    import numpy as np
    return np.load(os.path.join(GOLDEN, "multilevel_study.npz"))


@pytest.fixture(autouse=True)
def _fresh_cg_log(request):
    """GPU tests slice the per-solve CG log from a count they read themselves; the log keeps a
    bounded number of entries, so every GPU test starts from an empty one."""
    if request.node.get_closest_marker("gpu") is not None and gpu_available():
        from paper_2504_18526_b200.runtime import get_runtime
        get_runtime().reset_log()
    yield
