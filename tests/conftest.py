import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def stag_coords(dim, n, c):
    """Physical coordinates (x, y[, z]) of MAC location c (c < dim: velocity component
    c on its faces; c == dim: cell centres), as arrays indexed [j][i] / [k][j][i]
    (PAPER.md:419-438)."""
    h = 1.0 / n
    ax = []
    for a in range(dim):
        off = 0.0 if a == c else 0.5
        ax.append((np.arange(n) + off) * h)
    if dim == 2:
        Y, X = np.meshgrid(ax[1], ax[0], indexing="ij")
        return X, Y
    Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return X, Y, Z


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O
