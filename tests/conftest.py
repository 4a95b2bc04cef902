"""Shared test configuration.

`-m "not gpu"`: oracle vs golden fixtures, host logic, C-ABI surface (CPU only).
`-m gpu`:       CUDA path vs oracle / golden fixtures through the C ABI.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def load_golden(name):
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    out = {k: g[k] for k in g.files}
    if "results" in out:
        out["results"] = json.loads(str(out["results"]))
    return out


def tag_to_mode(tag, p):
    """'dp' | 'mp:t' | 'dst:t' -> (mode, t)."""
    if tag == "dp":
        return "dp", p
    mode, t = tag.split(":")
    return mode, int(t)


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_05324_b200 as mt  # noqa: F401
    from paper_2003_05324_b200 import _lib
    _lib.load()
    return torch
