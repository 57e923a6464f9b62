"""Dataset ingestion (container.py:91-189): a
class-subfolder image tree packed into a reference-format container,
byte-identical to the reference's ``build_container`` for the same
``BuildSpec``.

Per image: Pillow decode + EXIF orientation + RGB (the reference's own
loader, container.py:110-120), the downscale to ``max_resolution``
(fit_to_resolution, container.py:123-134) on the GPU through the bit-exact
``essl_resize_u8`` kernel (imgops.resize_bilinear), and the baseline
encoder (codec.py:574-632) in host C++ (essl_encode_jpeg, byte-identical
float64 FDCT).  Images are prepared by a thread pool and written strictly in
source order, so builds are byte-deterministic.
"""

from __future__ import annotations

import os
import struct
import zlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .container import (_HEADER_FMT, MAGIC, PAYLOAD_ALIGNMENT, RECORD_DTYPE, TABLE_ALIGNMENT,
                        VERSION, encode_jpeg)
from .errors import CroploadError

IMAGE_EXTENSIONS = {".jpg", ".jpeg", ".png", ".bmp", ".ppm", ".webp"}  # container.py:53


@dataclass(frozen=True)
class BuildSpec:
    """What to pack: a class-subfolder image tree plus compression knobs
    (container.py:68-82)."""

    source: str | Path
    max_resolution: int
    quality: int
    seed: int = 0

    def __post_init__(self):
        if self.max_resolution < 64:
            raise ValueError("max_resolution must be >= 64")
        if not 1 <= self.quality <= 100:
            raise ValueError("quality must be in [1, 100]")


@dataclass(frozen=True)
class BuildSummary:
    sample_count: int
    total_bytes: int


def scan_source_tree(source: str | Path) -> tuple[list[tuple[Path, int]], list[str]]:
    """Class subfolders in lexicographic order -> contiguous label ids
    (container.py:91-107)."""
    root = Path(source)
    if not root.is_dir():
        raise CroploadError(f"source directory not found: {root}")
    classes = sorted(p.name for p in root.iterdir() if p.is_dir())
    if not classes:
        raise CroploadError(f"no class subfolders in {root}")
    files: list[tuple[Path, int]] = []
    for label, name in enumerate(classes):
        for f in sorted((root / name).iterdir()):
            if f.is_file() and f.suffix.lower() in IMAGE_EXTENSIONS:
                files.append((f, label))
    if not files:
        raise CroploadError(f"no images found under {root}")
    return files, classes


def load_source_image(path: Path) -> np.ndarray:
    """Pillow decode, EXIF orientation applied, RGB (container.py:110-120)."""
    from PIL import Image, ImageOps
    try:
        with Image.open(path) as im:
            im = ImageOps.exif_transpose(im)
            return np.asarray(im.convert("RGB"))
    except CroploadError:
        raise
    except Exception as exc:
        raise CroploadError(f"cannot read source image {path}: {exc}") from exc


def fit_size(h: int, w: int, max_resolution: int) -> tuple[int, int]:
    """Output (h, w) of fit_to_resolution (container.py:123-134)."""
    if max(h, w) <= max_resolution:
        return h, w
    if w >= h:
        return max(1, int(h * max_resolution / w + 0.5)), max_resolution
    return max_resolution, max(1, int(w * max_resolution / h + 0.5))


def fit_to_resolution(img: np.ndarray, max_resolution: int, device=None) -> np.ndarray:
    """Downscale so max(side) <= max_resolution, never upscale; the resize
    runs on the GPU (bit-exact resize_bilinear, imgops.py:24-72)."""
    from .imgops import resize_bilinear
    h, w = img.shape[:2]
    oh, ow = fit_size(h, w, max_resolution)
    if (oh, ow) == (h, w):
        return img
    return resize_bilinear(img, oh, ow, device=device)


def build_container(spec: BuildSpec, out_path: str | Path, workers: int | None = None,
                    device=None) -> BuildSummary:
    """Pack a source tree into a container file (container.py:137-189)."""
    files, _ = scan_source_tree(spec.source)
    workers = workers or os.cpu_count() or 1

    def prepare(item):
        path, label = item
        img = fit_to_resolution(load_source_image(path), spec.max_resolution, device)
        return encode_jpeg(img, spec.quality), img.shape[1], img.shape[0], label

    n = len(files)
    table_size = n * RECORD_DTYPE.itemsize
    payload_base = -(-(TABLE_ALIGNMENT + table_size) // TABLE_ALIGNMENT) * TABLE_ALIGNMENT
    records = np.zeros(n, RECORD_DTYPE)
    out_path = Path(out_path)
    try:
        out = open(out_path, "wb")
    except OSError as exc:
        raise CroploadError(f"cannot write container {out_path}: {exc}") from exc
    with out:
        out.truncate(payload_base)
        out.seek(payload_base)
        pos = payload_base
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for i, (payload, w, h, label) in enumerate(pool.map(prepare, files, chunksize=4)):
                pad = -pos % PAYLOAD_ALIGNMENT
                if pad:
                    out.write(b"\x00" * pad)
                    pos += pad
                records[i] = (pos, len(payload), w, h, label, zlib.crc32(payload))
                out.write(payload)
                pos += len(payload)
        total = pos
        out.seek(0)
        out.write(struct.pack(_HEADER_FMT, MAGIC, VERSION, 0, n, TABLE_ALIGNMENT, payload_base,
                              spec.max_resolution, spec.quality, 0, TABLE_ALIGNMENT, spec.seed))
        out.seek(TABLE_ALIGNMENT)
        out.write(records.tobytes())
    return BuildSummary(n, total)
