"""Helpers shared by the test modules (imported as a top-level module:
pytest puts tests/ on sys.path)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def rel_block_err(a, b):
    """per block d: max|a_d - b_d| / max|b_d|."""
    out = []
    for d in range(b.shape[0]):
        m = np.abs(b[d]).max()
        out.append(np.abs(a[d] - b[d]).max() / m if m > 0 else np.abs(a[d]).max())
    return np.array(out)
