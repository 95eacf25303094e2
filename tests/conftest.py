"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with -m gpu);
everything else runs on the CPU (oracle vs golden fixtures, host logic, ABI
symbol checks, multi-process gloo tests).
"""

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def load_golden(name):
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("golden_small.npz")


@pytest.fixture(scope="session")
def golden_components():
    return load_golden("golden_components.npz")


@pytest.fixture(scope="session")
def golden_baseline():
    d = load_golden("golden_baseline.npz")
    d.update(load_golden("golden_c4.npz"))
    return d


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
