"""The packed dataset file (reference format, cropload/container.py:1-20).

Read side mirrors ``ContainerHandle`` (container.py:192-265); the GPU loader
additionally uploads the file once into HBM (``to_device``) so batches are
decoded from resident compressed bytes, or stages payloads per batch through
pinned memory (``essl_stage``).

Write side: ``write_container`` packs given payloads byte-for-byte in the
reference layout (container.py:137-189), ``build_synthetic`` makes benchmark
datasets with the native encoder (include/essl.h essl_encode_jpeg) and
``build_alias`` writes the epoch-scale cfg5 container whose records alias a
pool of distinct payloads.
"""

from __future__ import annotations

import ctypes
import mmap
import os
import struct
import zlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import CorruptionError, CroploadError, FormatError

MAGIC = b"ESSL"
VERSION = 1
TABLE_ALIGNMENT = 4096
PAYLOAD_ALIGNMENT = 64
_HEADER_FMT = "<4sHHQQQHBBIQ"
_HEADER_SIZE = struct.calcsize(_HEADER_FMT)  # 48

RECORD_DTYPE = np.dtype({
    "names": ["payload_offset", "payload_length", "width", "height", "label", "checksum"],
    "formats": ["<u8", "<u4", "<u2", "<u2", "<u4", "<u4"],
})
assert RECORD_DTYPE.itemsize == 24


@dataclass(frozen=True)
class ContainerHeader:
    magic: bytes
    version: int
    sample_count: int
    sample_table_offset: int
    payload_offset: int
    max_resolution: int
    quality: int
    alignment: int
    build_seed: int


class ContainerHandle:
    """Open container: validated header, record table, mmap'd payloads
    (container.py:192-247).  Thread-safe random reads."""

    def __init__(self, path: str | Path):
        self.path = Path(path)
        if not self.path.is_file():
            raise CroploadError(f"container not found: {self.path}")
        self._file = open(self.path, "rb")
        self._dev = {}
        self._pinned = None
        try:
            self._size = os.fstat(self._file.fileno()).st_size
            head = self._file.read(_HEADER_SIZE)
            if len(head) < _HEADER_SIZE:
                raise CorruptionError(f"{self.path}: file shorter than header")
            (magic, version, _, count, table_off, payload_off, max_res, quality, _,
             alignment, seed) = struct.unpack(_HEADER_FMT, head)
            if magic != MAGIC:
                raise FormatError(f"{self.path}: bad magic {magic!r}")
            if version != VERSION:
                raise FormatError(f"{self.path}: unsupported version {version}")
            if alignment == 0 or table_off % alignment or payload_off % alignment:
                raise FormatError(f"{self.path}: misaligned section offsets")
            if not 1 <= quality <= 100 or max_res < 64:
                raise FormatError(f"{self.path}: implausible header fields")
            table_end = table_off + count * RECORD_DTYPE.itemsize
            if table_end > self._size or payload_off < table_end:
                raise CorruptionError(f"{self.path}: truncated sample table")
            self.header = ContainerHeader(magic, version, count, table_off, payload_off,
                                          max_res, quality, alignment, seed)
            self._file.seek(table_off)
            raw = self._file.read(count * RECORD_DTYPE.itemsize)
            self.records = np.frombuffer(raw, RECORD_DTYPE)
            self._mmap = mmap.mmap(self._file.fileno(), 0, access=mmap.ACCESS_READ) \
                if self._size else None
            self.bytes = np.frombuffer(self._mmap, np.uint8) if self._mmap is not None \
                else np.zeros(0, np.uint8)
        except Exception:
            self._file.close()
            raise

    def __len__(self) -> int:
        return int(self.header.sample_count)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self) -> None:
        self._dev.clear()
        if getattr(self, "_pinned", None) is not None:
            if self._pinned[1] is None:
                from . import _native as N
                N.lib().essl_host_unregister(ctypes.c_void_p(self._pinned[0]))
            self._pinned = None
        self.bytes = None
        if getattr(self, "_mmap", None) is not None:
            try:
                self._mmap.close()
            except BufferError:  # a numpy view is still alive somewhere
                pass
            self._mmap = None
        self._file.close()

    def validate_index(self, index: int) -> tuple[int, int]:
        """Bounds/alignment checks of read_sample (container.py:251-262)."""
        if not 0 <= index < len(self):
            raise IndexError(f"sample index {index} out of range [0, {len(self)})")
        rec = self.records[index]
        off = int(rec["payload_offset"])
        length = int(rec["payload_length"])
        if off % PAYLOAD_ALIGNMENT:
            raise CorruptionError(f"sample {index}: misaligned payload")
        if off + length > self._size:
            raise CorruptionError(f"sample {index}: payload extends past end of file "
                                  f"(truncated container?)")
        return off, length

    def read_sample(self, index: int) -> tuple[bytes, int, int, int]:
        """-> (jpeg bytes, width, height, label); CRC-verified on the host
        (container.py:249-265).  The GPU loader verifies CRCs on device."""
        off, length = self.validate_index(index)
        rec = self.records[index]
        payload = self._mmap[off:off + length]
        if zlib.crc32(payload) != int(rec["checksum"]):
            raise CorruptionError(f"sample {index}: checksum mismatch")
        return payload, int(rec["width"]), int(rec["height"]), int(rec["label"])

    def validate_all(self) -> None:
        """Vectorised bounds/alignment check of every record (raises like
        read_sample would on first use)."""
        offs = self.records["payload_offset"].astype(np.uint64)
        lens = self.records["payload_length"].astype(np.uint64)
        bad = np.nonzero((offs % PAYLOAD_ALIGNMENT != 0) | (offs + lens > self._size))[0]
        if bad.size:
            self.validate_index(int(bad[0]))

    def to_device(self, device):
        """The whole file as a uint8 CUDA tensor (HBM-resident dataset);
        record offsets index it directly.  Cached per device."""
        import torch
        key = str(device)
        t = self._dev.get(key)
        if t is None:
            import warnings
            with warnings.catch_warnings():  # read-only mmap: the copy never writes it
                warnings.simplefilter("ignore", UserWarning)
                host = torch.frombuffer(self._mmap, dtype=torch.uint8) if self._size else \
                    torch.zeros(1, dtype=torch.uint8)
            t = torch.empty(max(self._size, 1), dtype=torch.uint8, device=device)
            chunk = 1 << 28
            for s in range(0, self._size, chunk):
                t[s:s + chunk].copy_(host[s:s + chunk], non_blocking=False)
            self._dev[key] = t
        return t

    def pinned_host(self) -> int:
        """Host address of the whole file, page-locked for copy-engine
        gathers (essl_stage_pinned): the read-only file mapping registered in
        place, or (where the driver refuses that) a pinned copy."""
        if self._pinned is not None:
            return self._pinned[2]
        from . import _native as N
        import torch
        torch.cuda.init()
        base = int(self.bytes.ctypes.data) if self._size else 0
        if self._size and N.lib().essl_host_register(ctypes.c_void_p(base), self._size, 1) == 0:
            host, buf = base, None
        else:
            buf = torch.empty(max(self._size, 1), dtype=torch.uint8, pin_memory=True)
            if self._size:
                buf.numpy()[:self._size] = self.bytes
            host = int(buf.data_ptr())
        dev = ctypes.c_void_p()
        N.check(N.lib().essl_host_device_ptr(ctypes.c_void_p(host), ctypes.byref(dev)),
                "essl_host_device_ptr")
        self._pinned = (host, buf, int(dev.value))
        return self._pinned[2]

    def max_dims(self) -> tuple[int, int]:
        if len(self) == 0:
            return 1, 1
        return int(self.records["width"].max()), int(self.records["height"].max())

    def max_payload(self) -> int:
        return int(self.records["payload_length"].max()) if len(self) else 4


def open_container(path: str | Path) -> ContainerHandle:
    return ContainerHandle(path)


def verify_crcs(path: str | Path) -> list[int]:
    """Indices of samples failing checksum or bounds (container.py:270-281)."""
    bad = []
    with open_container(path) as h:
        for i in range(len(h)):
            try:
                h.read_sample(i)
            except CorruptionError:
                bad.append(i)
    return bad


# ---------------------------------------------------------------------------
# writers

def write_container(out_path: str | Path, payloads: list[bytes], widths, heights, labels,
                    max_resolution: int, quality: int, seed: int = 0,
                    record_payload: np.ndarray | None = None) -> int:
    """Pack payloads in the reference layout (container.py:137-189): header,
    24-byte records at 4096, payloads 64-byte aligned from the next 4096
    boundary.  ``record_payload`` (optional int array, one entry per record)
    makes records alias payloads (the cfg5 epoch-scale stream).  Returns the
    file size."""
    n_pay = len(payloads)
    rp = np.arange(n_pay) if record_payload is None else np.asarray(record_payload, np.int64)
    n = len(rp)
    table_size = n * RECORD_DTYPE.itemsize
    payload_base = -(-(TABLE_ALIGNMENT + table_size) // TABLE_ALIGNMENT) * TABLE_ALIGNMENT
    offs = np.zeros(n_pay, np.uint64)
    crcs = np.zeros(n_pay, np.uint32)
    with open(out_path, "wb") as out:
        out.truncate(payload_base)
        out.seek(payload_base)
        pos = payload_base
        for i, p in enumerate(payloads):
            pad = -pos % PAYLOAD_ALIGNMENT
            if pad:
                out.write(b"\x00" * pad)
                pos += pad
            offs[i] = pos
            crcs[i] = zlib.crc32(p)
            out.write(p)
            pos += len(p)
        records = np.zeros(n, RECORD_DTYPE)
        records["payload_offset"] = offs[rp]
        records["payload_length"] = np.array([len(p) for p in payloads], np.uint32)[rp]
        records["width"] = np.asarray(widths, np.uint16)[rp] if len(widths) == n_pay else widths
        records["height"] = np.asarray(heights, np.uint16)[rp] if len(heights) == n_pay else heights
        records["label"] = np.asarray(labels, np.uint32) if len(labels) == n else \
            np.asarray(labels, np.uint32)[rp]
        records["checksum"] = crcs[rp]
        out.seek(0)
        out.write(struct.pack(_HEADER_FMT, MAGIC, VERSION, 0, n, TABLE_ALIGNMENT, payload_base,
                              max_resolution, quality, 0, TABLE_ALIGNMENT, seed))
        out.seek(TABLE_ALIGNMENT)
        out.write(records.tobytes())
    return pos


def encode_jpeg(image: np.ndarray, quality: int, restart_interval: int = 0) -> bytes:
    """Baseline 4:2:0 encoder (codec.py:574-632), native host C++."""
    from . import _native as N
    img = np.ascontiguousarray(image, dtype=np.uint8)
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError(f"expected (h, w, 3) RGB image, got {img.shape}")
    h, w = img.shape[:2]
    if h < 1 or w < 1:
        raise ValueError("image dimensions must be >= 1")
    if not 1 <= quality <= 100:
        raise ValueError(f"quality must be in [1, 100], got {quality}")
    mcus = -(-w // 16) * -(-h // 16)
    cap = 6 * mcus * 450 + 4096 + (2 * (mcus // restart_interval + 1) if restart_interval else 0)
    out = np.empty(cap, np.uint8)
    n = N.lib().essl_encode_jpeg(N.ptr(img), h, w, quality, restart_interval, N.ptr(out), cap)
    if n < 0:
        raise RuntimeError(f"essl_encode_jpeg failed ({n})")
    return out[:n].tobytes()


def synth_image(seed: int, height: int, width: int) -> np.ndarray:
    """Deterministic synthetic natural-style RGB image (own generator)."""
    from . import _native as N
    out = np.empty((height, width, 3), np.uint8)
    N.check(N.lib().essl_synth_image(seed & (2**64 - 1), height, width, N.ptr(out)),
            "essl_synth_image")
    return out


def build_synthetic(out_path: str | Path, n_images: int, side: int | tuple[int, int],
                    quality: int, classes: int = 4, seed: int = 1,
                    workers: int | None = None, n_records: int | None = None,
                    restart_interval: int = 0) -> dict:
    """Synthetic benchmark container: ``n_images`` distinct payloads of
    side x side (or a (min, max) side range) at ``quality``.  With
    ``n_records`` > n_images the record table aliases the pool (cfg5).
    ``restart_interval`` > 0 writes DRI + RSTn every that many MCUs (the
    opt-in restart-marker variant; not byte-identical to
    the reference builder's output, which has no restarts)."""
    lo, hi = (side, side) if isinstance(side, int) else side
    rng = np.random.default_rng(seed)
    dims = [(int(rng.integers(lo, hi + 1)), int(rng.integers(lo, hi + 1))) for _ in range(n_images)]

    def make(i):
        h, w = dims[i]
        return encode_jpeg(synth_image(seed * 1_000_003 + i, h, w), quality, restart_interval)

    with ThreadPoolExecutor(max_workers=workers or os.cpu_count() or 1) as pool:
        payloads = list(pool.map(make, range(n_images)))
    widths = [d[1] for d in dims]
    heights = [d[0] for d in dims]
    n = n_records or n_images
    rp = np.arange(n) % n_images
    labels = (np.arange(n) % classes).astype(np.uint32)
    size = write_container(out_path, payloads, widths, heights, labels, max(hi, 64), quality,
                           seed, record_payload=rp)
    return {"path": str(out_path), "records": n, "distinct": n_images, "bytes": size,
            "mean_payload": float(np.mean([len(p) for p in payloads]))}
