"""Batch stream wire format (cli.py:132-211): framing on
the CPU (a stand-in loader with the golden configuration's shapes reproduces
the reference stream's header and first frame byte for byte), and the whole
stream from the GPU loader against the reference's stream (SHA-256) and its
--digest lines."""

from __future__ import annotations

import io
import json
import subprocess
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

GS = json.loads((GOLDEN / "golden_stream.json").read_text())


class _FakeLoader:
    """Shapes of the golden configuration (16 samples, batch 16, res 96, k 27)."""

    def __init__(self, n=16, b=16, res=96, k=27):
        self.config = SimpleNamespace(out_dtype="float32", batch_size=b, res=res)
        self.mask_spec = SimpleNamespace(masked_count=k)
        self.n, self.b, self.res, self.k = n, b, res, k
        self.batches_per_epoch = -(-n // b)

    def __len__(self):
        return self.n

    def epoch(self, e):
        rng = np.random.default_rng(e)
        for s in range(0, self.n, self.b):
            yield _Batch(rng, min(self.b, self.n - s), s, self.res, self.k, e)


class _Batch:
    def __init__(self, rng, b, s, res, k, e):
        self.pixels = rng.standard_normal((b, 3, res, res)).astype(np.float32)
        self.labels = np.arange(b, dtype=np.int64)
        self.indices = np.arange(s, s + b, dtype=np.int64)
        self.mask = np.tile(np.arange(k, dtype=np.int32), (b, 1))
        self.epoch = e

    def __len__(self):
        return len(self.labels)


def test_stream_framing_matches_reference_head():
    from paper_2404_00509_b200.stream import read_stream, write_stream
    for run in GS["runs"]:
        buf = io.BytesIO()
        n = write_stream(_FakeLoader(), run["epoch"], buf, run["batches"])
        raw = buf.getvalue()
        assert n == len(raw) == run["bytes"]
        assert raw[:256].hex() == run["head"]
        header, batches = read_stream(raw)
        assert header["batches"] == len(batches) == 1
        assert header["mask_k"] == 27 and header["pixel_dtype"] == "float32"
        for meta, arrays in batches:
            assert arrays["pixels"].size == meta["b"] * 3 * 96 * 96
            assert arrays["mask"].size == meta["b"] * 27
    with pytest.raises(ValueError):
        read_stream(raw[:-3])
    with pytest.raises(ValueError):
        read_stream(b"XXXXXXXX" + raw[8:])


@pytest.mark.gpu
def test_gpu_stream_equals_reference_stream(tmp_path, cuda):
    cfg = dict(GS["config"], data=str(GOLDEN / GS["config"]["data"]))
    (tmp_path / "cfg.json").write_text(json.dumps(cfg))
    import hashlib
    for run in GS["runs"]:
        base = [sys.executable, "-m", "paper_2404_00509_b200", "stream", "--config",
                str(tmp_path / "cfg.json"), "--epoch", str(run["epoch"]), "--batches",
                str(run["batches"])]
        raw = subprocess.run(base, capture_output=True, check=True, cwd=ROOT).stdout
        assert len(raw) == run["bytes"]
        assert hashlib.sha256(raw).hexdigest() == run["sha256"]
        dig = subprocess.run(base + ["--digest"], capture_output=True, check=True, text=True,
                             cwd=ROOT).stdout
        assert [json.loads(x) for x in dig.strip().splitlines()] == run["digests"]
