"""Exception hierarchy (mirrors cropload/errors.py:4-31) and the mapping from
per-image device status codes (include/essl.h ESSL_ST_*) to exceptions with
the reference's messages (codec.py, container.py)."""

from __future__ import annotations


class CroploadError(Exception):
    """Base class for all errors raised by this package (errors.py:4-5)."""


class FormatError(CroploadError):
    """A file is not a valid container (errors.py:8-9)."""


class CorruptionError(CroploadError):
    """Stored data failed an integrity check (errors.py:12-13)."""


class DecodeError(CroploadError):
    """A JPEG stream could not be decoded (errors.py:16-27)."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (at byte offset {offset})"
        super().__init__(message)
        self.offset = offset


class ConfigError(CroploadError):
    """A configuration document or argument violates its schema (errors.py:30-31)."""


class UnsupportedStreamError(DecodeError):
    """Streams outside the GPU decoder's limits (hostile streams only:
    coefficients outside int16, more than 64 scans / 24 Huffman tables)."""


ST_OK, ST_CORRUPT_HUFFMAN, ST_MISSING_RST, ST_TRUNCATED = 0, 1, 3, 4
ST_CRC, ST_UNSUPPORTED, ST_RECT, ST_MALFORMED = 5, 6, 7, 8
ST_HUFFTABLE, ST_QUANT, ST_CAPACITY = 9, 10, 11

# (message, carries offset) per reason code, codec.py:104-330
_REASONS = {
    1: ("not a JPEG stream (missing SOI)", True),
    2: ("expected marker", True),
    3: ("unexpected end of stream", True),
    4: ("truncated marker segment", True),
    5: ("truncated DQT", True),
    6: ("truncated DHT", True),
    7: ("multiple SOF markers", True),
    8: ("unsupported precision", True),
    9: ("zero image dimension", True),
    10: ("unsupported component count", True),
    11: ("unsupported sampling", True),
    12: ("unsupported SOF type (not sequential/progressive Huffman)", True),
    13: ("SOS before SOF", True),
    14: ("scan references unknown component", True),
    15: ("no image data found", True),
    16: ("restart marker without DRI", True),
    17: ("too many restart markers", True),
    18: ("progressive JPEG is not supported by the GPU decoder", False),
    19: ("multi-scan / partially interleaved JPEG is not supported by the GPU decoder", False),
    20: ("scan references undefined Huffman table", False),
    21: ("invalid Huffman table (code overflow)", False),
    22: ("Huffman table with more than 256 symbols", False),
    23: ("marker segment shorter than its fields", True),
    24: ("coefficient out of int16 range", False),
    25: ("image exceeds the context scratch capacity", False),
    26: ("progressive DC scan with Se != 0", False),
    27: ("progressive AC scan must be single-component", False),
    28: ("partially interleaved scans are not supported", False),
    29: ("too many scans or Huffman tables for the GPU decoder", False),
}


def status_error(status: int, reason: int = 0, offset: int = -1, *,
                 sample: int | None = None, rect=None, dims=None) -> Exception:
    """Exception for a nonzero per-image status."""
    off = None if offset is None or offset < 0 else int(offset)
    if status == ST_CRC:
        who = f"sample {sample}" if sample is not None else "payload"
        return CorruptionError(f"{who}: checksum mismatch")
    if status == ST_RECT:
        return ValueError(f"crop rect {rect} out of bounds for "
                          f"{dims[0]}x{dims[1]} image" if dims else f"crop rect {rect} out of bounds")
    if status == ST_CORRUPT_HUFFMAN:
        exc = DecodeError("corrupt entropy-coded data", off)
    elif status == ST_MISSING_RST:
        exc = DecodeError("missing restart marker", off)
    elif status == ST_TRUNCATED:
        exc = DecodeError("truncated entropy-coded data", off)
    elif status == ST_QUANT:
        exc = DecodeError(f"missing quantization table {offset}")
    elif status == ST_UNSUPPORTED:
        msg, _ = _REASONS.get(reason, ("unsupported stream", False))
        exc = UnsupportedStreamError(msg)
    elif status in (ST_MALFORMED, ST_HUFFTABLE):
        msg, with_off = _REASONS.get(reason, ("malformed stream", True))
        exc = DecodeError(msg, off if with_off else None)
    elif status == ST_CAPACITY:
        exc = CroploadError(_REASONS[25][0])
    else:
        exc = DecodeError(f"decode failed with status {status}", off)
    if sample is not None and isinstance(exc, DecodeError):
        exc.sample = sample
    return exc
