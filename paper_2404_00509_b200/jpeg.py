"""Codec operator API on the GPU (mirror of cropload/jpeg: codec.py:43-71,
434-511).  ``decode_crop`` / ``decode_full`` run the sm_100a decoder
(k_decode + k_crop_u8); ``encode_jpeg`` is the native host encoder."""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .container import encode_jpeg  # noqa: F401  (re-export, codec.py:574)
from .engine import default_engine
from .errors import DecodeError, status_error


@dataclass(frozen=True)
class CropRect:
    """Pixel-space crop window (codec.py:43-56)."""

    x: int
    y: int
    w: int
    h: int

    def validate(self, width: int, height: int) -> None:
        if self.w < 1 or self.h < 1 or self.x < 0 or self.y < 0 \
                or self.x + self.w > width or self.y + self.h > height:
            raise ValueError(f"crop rect {self} out of bounds for {width}x{height} image")


@dataclass
class DecodeStats:
    """Work counters (codec.py:59-71).  fallback_full: a multi-scan
    (progressive) stream took the full decode of every scan, as in the
    reference (codec.py:461-469) -- on the GPU too."""

    mcus_entropy_decoded: int
    mcus_reconstructed: int
    fallback_full: bool = False


def peek_dims(data: bytes) -> tuple[int, int] | None:
    """(width, height) from the first SOF0/1/2 segment, or None.  Only used
    to size decode_full's output; the GPU parser is authoritative."""
    pos, n = 2, len(data)
    if n < 4 or data[0] != 0xFF or data[1] != 0xD8:
        return None
    while pos + 4 <= n:
        if data[pos] != 0xFF:
            return None
        while pos < n and data[pos] == 0xFF:
            pos += 1
        if pos >= n:
            return None
        m = data[pos]
        pos += 1
        if m == 0xD9 or m == 0xDA:
            return None
        if m == 0x01 or 0xD0 <= m <= 0xD7:
            continue
        if pos + 2 > n:
            return None
        seglen = struct.unpack_from(">H", data, pos)[0]
        if m in (0xC0, 0xC1, 0xC2) and pos + 7 <= n:
            h, w = struct.unpack_from(">HH", data, pos + 3)
            return w, h
        pos += seglen
    return None


def decode_crops(items: list[tuple[bytes, CropRect]], device=None):
    """Batched decode_crop: [(bytes, rect)] -> [(rgb uint8 [h,w,3], stats)]."""
    import torch
    eng = default_engine(device)
    n = len(items)
    if n == 0:
        return []
    lens = np.array([len(d) for d, _ in items], np.uint32)
    offs = np.zeros(n, np.uint64)
    offs[1:] = np.cumsum((lens.astype(np.uint64) + 63) // 64 * 64)[:-1]
    blob = np.zeros(int(offs[-1] + ((int(lens[-1]) + 63) // 64 * 64) + 64), np.uint8)
    for i, (d, _) in enumerate(items):
        blob[int(offs[i]):int(offs[i]) + len(d)] = np.frombuffer(d, np.uint8)
    dblob = torch.from_numpy(blob).to(eng.device)
    samples = eng.samples(n)
    samples["offset"] = offs
    samples["length"] = lens
    out_off = np.zeros(n, np.uint64)
    acc = 0
    for i, (_, r) in enumerate(items):
        samples[i]["x"], samples[i]["y"], samples[i]["w"], samples[i]["h"] = r.x, r.y, r.w, r.h
        out_off[i] = acc
        acc += max(r.w, 0) * max(r.h, 0) * 3
    out = torch.empty(max(acc, 1), dtype=torch.uint8, device=eng.device)
    res = eng.new_results(n)
    max_side = max(max(r.x + r.w, r.y + r.h) for _, r in items)
    eng.decode_crop_u8(dblob.data_ptr(), samples, out, out_off, results=res,
                       max_side=max(max_side, 16))
    host = out.cpu().numpy()
    rh = res.cpu().numpy()
    outs = []
    for i, (_, r) in enumerate(items):
        if rh[i, 0] != 0:
            raise status_error(int(rh[i, 0]), int(rh[i, 1]), int(rh[i, 2]),
                               rect=r, dims=(int(rh[i, 5]), int(rh[i, 6])))
        o = int(out_off[i])
        rgb = host[o:o + r.w * r.h * 3].reshape(r.h, r.w, 3).copy()
        outs.append((rgb, DecodeStats(int(rh[i, 3]), int(rh[i, 4]), bool(rh[i, 1] == 1))))
    return outs


def decode_crop(data: bytes, rect: CropRect, device=None):
    """Decode only the MCUs needed for ``rect`` (codec.py:448-511) on the GPU."""
    return decode_crops([(bytes(data), rect)], device)[0]


def decode_full(data: bytes, device=None):
    """Whole-image decode (codec.py:434-445) == full-rect crop decode (its
    stats never flag the fallback, as the reference's decode_full)."""
    dims = peek_dims(bytes(data))
    rect = CropRect(0, 0, dims[0], dims[1]) if dims else CropRect(0, 0, 1, 1)
    if dims is None or dims[0] == 0 or dims[1] == 0:
        # let the GPU parser produce the reference's error
        try:
            decode_crops([(bytes(data), rect)], device)
        except ValueError as exc:
            raise DecodeError(str(exc)) from exc
        raise DecodeError("no image data found")
    rgb, st = decode_crops([(bytes(data), rect)], device)[0]
    return rgb, DecodeStats(st.mcus_entropy_decoded, st.mcus_reconstructed, False)
