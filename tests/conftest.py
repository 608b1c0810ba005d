import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    return load


def mapping_submaps(g):
    """Dense submaps + reference global poses from tests/golden/mapping.npz."""
    n = int(g["n_submaps"])
    sms, globs = [], []
    for j in range(n):
        sms.append(dict(depth=g[f"sm{j}_depth"], conf=g[f"sm{j}_conf"],
                        frame_ids=g[f"sm{j}_frame_ids"], pose_q=g[f"sm{j}_pose_q"],
                        pose_t=g[f"sm{j}_pose_t"], K=g[f"sm{j}_K"]))
        globs.append((float(g[f"sm{j}_gs"]), g[f"sm{j}_gq"], g[f"sm{j}_gt"]))
    return sms, globs
