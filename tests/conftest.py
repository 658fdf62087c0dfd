"""Shared test setup.

Markers: ``gpu`` = needs a CUDA device (run on the B200 box with -m gpu).
The CPU oracle (oracle/, test infrastructure) is built on demand.
"""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

MASTER = 20250814


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"golden fixture {name} not generated")
    return json.loads(path.read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def hex_to_spins(h, n):
    import numpy as np

    hh = h + ("0" if len(h) % 2 else "")
    bits = np.unpackbits(np.frombuffer(bytes.fromhex(hh), np.uint8))[:n]
    return np.where(bits == 1, 1, -1).astype(np.int8)
