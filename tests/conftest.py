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


def pytest_sessionfinish(session, exitstatus):
    """With a bounds-checked library (ESSL_CHECKED build selected through
    ESSL_LIB), fail the run if any device-side bounds check fired; the
    counters are written to gpurun_out/bounds_check.json."""
    import os
    if not os.environ.get("ESSL_LIB", "").endswith("checked/libessl.so"):
        return
    try:
        import torch
        if not torch.cuda.is_available():
            return
        from paper_2404_00509_b200 import _native as N
        out = np.zeros(16, np.uint32)
        rc = N.lib().essl_check_read(N.ptr(out), 16, 0)
    except Exception as exc:  # (reported, not raised from a hook)
        print(f"bounds check read failed: {exc}")
        return
    names = ["list", "coef", "ms_coef", "plane", "clean", "src", "out", "ckpt"]
    res = {"checked_build": rc == 1, "violations": {n: int(out[i]) for i, n in enumerate(names)}}
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "bounds_check.json").write_text(json.dumps(res, indent=1))
    print("bounds check:", res)
    if rc != 1 or int(out.sum()) != 0:
        session.exitstatus = 1
