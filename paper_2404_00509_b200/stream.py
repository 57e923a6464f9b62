"""Batch stream wire format: the binary frames the
reference's ``cropload stream`` command writes for its bindings frontend
(cli.py:132-211, frontend/src/wire.ts), fed here by the GPU loader.

Layout (little endian), byte-identical to the reference for the same loader
configuration:

    b"CLDSTRM1"
    u32 len | header JSON {version, batches, samples, batch_size, res, epoch,
                           mask_k, pixel_dtype} | spaces to 8-byte alignment
    per batch:
      u32 len | meta JSON {batch, b, epoch, mask_k, payload, pixels, labels,
                           indices, mask}  ([offset, length] in the payload)
      payload: pixels float32 [b,3,res,res] | labels int64 [b] |
               indices int64 [b] | mask int32 [b,k] | zeros to 8 bytes
    b"CLDEND00"

``--digest`` mode writes one JSON line of SHA-256 digests per batch instead
(cli.py:147-162).  Batches come off the GPU through pinned host buffers
while the loader keeps decoding the next ones.
"""

from __future__ import annotations

import hashlib
import io
import json
import struct
from pathlib import Path

import numpy as np

from .errors import ConfigError

STREAM_MAGIC = b"CLDSTRM1"  # cli.py:29
STREAM_END = b"CLDEND00"    # cli.py:30


def stream_meta(obj, written: int) -> bytes:
    """u32 length + compact JSON + spaces so the next byte is 8-aligned
    (cli.py:132-135; `written` = bytes already in the stream)."""
    raw = json.dumps(obj, separators=(",", ":")).encode()
    pad = -(4 + len(raw) + written) % 8
    return struct.pack("<I", len(raw) + pad) + raw + b" " * pad


def _host(t) -> np.ndarray:
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def _batches(loader, epoch: int, n_batches: int):
    for bi, batch in enumerate(loader.epoch(epoch)):
        if bi >= n_batches:
            break
        yield bi, batch


def _check(loader) -> tuple[int, int]:
    import torch
    if loader.config.out_dtype != "float32":
        raise ConfigError("the batch stream carries float32 pixels (pixel_dtype); "
                          "use out_dtype='float32'")
    k = loader.mask_spec.masked_count if loader.mask_spec is not None else 0
    return k, torch.float32


def write_stream(loader, epoch: int, out, batches: int | None = None) -> int:
    """Write the binary stream of `batches` batches (default: the epoch) of
    `epoch` to the binary file object `out`; returns the bytes written."""
    mask_k, _ = _check(loader)
    cfg = loader.config
    n_batches = loader.batches_per_epoch if batches is None else min(loader.batches_per_epoch,
                                                                        batches)
    written = 0

    def emit(data: bytes):
        nonlocal written
        out.write(data)
        written += len(data)

    emit(STREAM_MAGIC)
    emit(stream_meta({"version": 1, "batches": n_batches, "samples": len(loader),
                      "batch_size": cfg.batch_size, "res": cfg.res, "epoch": epoch,
                      "mask_k": mask_k, "pixel_dtype": "float32"}, written))
    for bi, batch in _batches(loader, epoch, n_batches):
        pixels = _host(batch.pixels).tobytes()
        labels = _host(batch.labels).astype(np.int64, copy=False).tobytes()
        indices = _host(batch.indices).astype(np.int64, copy=False).tobytes()
        mask = _host(batch.mask).astype(np.int32, copy=False).tobytes() if batch.mask is not None else b""
        pad = (-len(mask)) % 8
        segs, off = {}, 0
        for name, blob in (("pixels", pixels), ("labels", labels), ("indices", indices),
                           ("mask", mask)):
            segs[name] = [off, len(blob)]
            off += len(blob)
        emit(stream_meta({"batch": bi, "b": len(batch), "epoch": int(batch.epoch),
                          "mask_k": mask_k, "payload": off + pad, **segs}, written))
        for blob in (pixels, labels, indices, mask):
            emit(blob)
        if pad:
            emit(b"\x00" * pad)
    emit(STREAM_END)
    return written


def digest_stream(loader, epoch: int, batches: int | None = None):
    """Per-batch SHA-256 digests (cli.py:147-162), one dict per batch."""
    mask_k, _ = _check(loader)
    n_batches = loader.batches_per_epoch if batches is None else min(loader.batches_per_epoch,
                                                                        batches)
    for bi, batch in _batches(loader, epoch, n_batches):
        yield {"batch": bi, "b": len(batch), "epoch": int(batch.epoch), "mask_k": mask_k,
               "pixels_sha256": hashlib.sha256(_host(batch.pixels).tobytes()).hexdigest(),
               "labels_sha256": hashlib.sha256(_host(batch.labels).tobytes()).hexdigest(),
               "indices_sha256": hashlib.sha256(_host(batch.indices).tobytes()).hexdigest(),
               "mask_sha256": (hashlib.sha256(_host(batch.mask).tobytes()).hexdigest()
                               if batch.mask is not None else None)}


def read_stream(raw) -> tuple[dict, list]:
    """Parse a stream (bytes or a path): (header, [(meta, {name: array})])
    with the checks of the reference's parser (test_cli.py:170-191)."""
    if isinstance(raw, (str, Path)):
        raw = Path(raw).read_bytes()
    buf = io.BytesIO(raw)

    def take(n):
        data = buf.read(n)
        if len(data) != n:
            raise ValueError("truncated stream")
        return data

    if take(8) != STREAM_MAGIC:
        raise ValueError("not a batch stream (bad magic)")
    (hlen,) = struct.unpack("<I", take(4))
    header = json.loads(take(hlen))
    batches = []
    for _ in range(header["batches"]):
        (mlen,) = struct.unpack("<I", take(4))
        meta = json.loads(take(mlen))
        if buf.tell() % 8:
            raise ValueError("payload not 8-aligned")
        payload = take(meta["payload"])
        arrays = {}
        for name, dt in (("pixels", np.float32), ("labels", np.int64), ("indices", np.int64),
                         ("mask", np.int32)):
            off, length = meta[name]
            arrays[name] = np.frombuffer(payload[off:off + length], dt)
        batches.append((meta, arrays))
    if take(8) != STREAM_END:
        raise ValueError("missing end marker")
    if buf.read():
        raise ValueError("trailing bytes after the end marker")
    return header, batches
