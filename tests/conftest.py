import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def dense_from_configs(configs, n_upps=4):
    """Per-job lists of (upp, g, R) -> dense int32 runtime[T][U][Gmax] (0 = infeasible)."""
    gmax = max(g for job in configs for _, g, _ in job)
    table = np.zeros((len(configs), n_upps, gmax), np.int32)
    for t, job in enumerate(configs):
        for u, g, r in job:
            table[t, u, g - 1] = r
    return table


def dense_from_single(jobs):
    """Per-job single configuration (g, R) under UPP 0 -> dense table."""
    return dense_from_configs([[(0, g, r)] for g, r in jobs], n_upps=1)


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
