"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def arrays():
    return dict(np.load(GOLDEN / "arrays.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def stream_bytes(name: str) -> bytes:
    return (GOLDEN / "streams" / f"{name}.jpg").read_bytes()


@pytest.fixture(scope="session")
def native():
    from paper_2404_00509_b200 import build
    build.build()
    from paper_2404_00509_b200 import _native
    return _native


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2404_00509_b200 import build
    build.build()
    return torch.device("cuda", 0)
