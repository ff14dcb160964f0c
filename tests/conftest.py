"""pytest configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here on the CPU box (oracle pins, host logic, ABI exports, gloo
multi-process tests); `-m gpu` runs on a B200 and calls the product path through the
C ABI (parity against the oracle).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product path")


def golden_rows(name):
    """Non-comment rows of tests/golden/<name>, split on whitespace."""
    path = os.path.join(ROOT, "tests", "golden", name)
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.lib()
    return O
