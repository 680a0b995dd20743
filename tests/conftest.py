import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")
DATA = os.path.join(ROOT, "data")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLD))


@pytest.fixture(scope="session")
def workloads():
    return dict(np.load(os.path.join(DATA, "workloads.npz")))


@pytest.fixture(scope="session")
def wfix():
    return dict(np.load(os.path.join(DATA, "w_fix.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle import snn_oracle
    return snn_oracle


@pytest.fixture(scope="session")
def oparams(oracle):
    return oracle.Params()


@pytest.fixture(scope="session")
def sd():
    import paper_1711_03637_b200 as sd
    return sd


@pytest.fixture(scope="session")
def toy():
    """oracle/gen_toy.py: the reference's two-class convergence corpus and its
    lateral-inhibition corpus, with the reference's own results."""
    return dict(np.load(os.path.join(os.path.dirname(GOLD), "toy_reference.npz")))


@pytest.fixture(scope="session")
def canvases():
    """oracle/gen_canvases.py: canvases of many shapes with the reference's
    preprocess_pipeline outputs (blank ones flagged)."""
    z = dict(np.load(os.path.join(os.path.dirname(GOLD), "canvases.npz")))
    z["list"] = [z["pixels"][o:o + h * w].reshape(h, w) for (h, w), o in zip(z["shapes"], z["offsets"][:-1])]
    return z
