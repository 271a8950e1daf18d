import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


class GoldenGrid:
    """Grid instance stored in a golden .npz (duck-types the reference GridEnergy)."""

    def __init__(self, d):
        self.dims = tuple(int(v) for v in d["dims"])
        self.connectivity = str(d["conn"])
        self.w = d["w"]
        self.dir_weights = [d["dw%d" % k] for k in range(4) if "dw%d" % k in d]
        self.n = self.w.size


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_grid(name):
    d = load_golden(name)
    return GoldenGrid(d), d


def aar_cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "aar_*.npz")))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle as orc
    orc.lib()
    return orc


def level_cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "levels_*.npz")))


def dual_cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "dual_*.npz")))
