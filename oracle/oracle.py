"""ctypes wrapper over the C oracle (oracle/essl_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs.  The product package never imports it.

Function names mirror the reference API they restate
(/root/reference/pkg/src/cropload/...), returning numpy arrays.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

# Status codes (shared with include/essl.h).
ST_OK, ST_CORRUPT_HUFFMAN, ST_MISSING_RST, ST_TRUNCATED = 0, 1, 3, 4
ST_CRC, ST_UNSUPPORTED, ST_RECT, ST_MALFORMED = 5, 6, 7, 8
ST_HUFFTABLE, ST_QUANT = 9, 10


class OracleError(Exception):
    def __init__(self, status, reason=0, offset=-1):
        super().__init__(f"oracle status {status} reason {reason} offset {offset}")
        self.status, self.reason, self.offset = int(status), int(reason), int(offset)


def build() -> Path:
    """Compile the oracle with its Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


class OrcLoaderCfg(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("epoch", ctypes.c_uint64),
                ("res", ctypes.c_int), ("scale_lo", ctypes.c_double),
                ("scale_hi", ctypes.c_double), ("ratio_lo", ctypes.c_double),
                ("ratio_hi", ctypes.c_double), ("mask_grid", ctypes.c_int),
                ("mask_k", ctypes.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        u64, i64, i32, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_rng_init.restype = u64
        L.orc_rng_init.argtypes = [u64, u64, u64, u64]
        L.orc_rng_next.restype = u64
        L.orc_rng_next.argtypes = [P]
        L.orc_rng_random.restype = dbl
        L.orc_rng_random.argtypes = [P]
        L.orc_rng_randint.restype = i64
        L.orc_rng_randint.argtypes = [P, i64]
        L.orc_epoch_permutation.argtypes = [u64, u64, i64, P]
        L.orc_sample_rrc.argtypes = [P, i64, i64, dbl, dbl, dbl, dbl, i32, P]
        L.orc_mask_count.restype = i32
        L.orc_mask_count.argtypes = [i32, dbl]
        L.orc_sample_mask.argtypes = [P, i32, i32, P]
        L.orc_crc32.restype = ctypes.c_uint32
        L.orc_crc32.argtypes = [P, ctypes.c_size_t]
        L.orc_destuff.restype = i32
        L.orc_destuff.argtypes = [P, i32, i32, P, P, i32, P, P]
        L.orc_idct_block.argtypes = [P, P, P, i32]
        L.orc_decode_crop.restype = i32
        L.orc_decode_crop.argtypes = [P, i32, i32, i32, i32, i32, i32, P, P, P]
        L.orc_jpeg_info.restype = i32
        L.orc_jpeg_info.argtypes = [P, i32, P, P]
        L.orc_dump_coefs.restype = i32
        L.orc_dump_coefs.argtypes = [P, i32, i32, i32, i32, i32, P, i64, P, P]
        L.orc_resize_bilinear.argtypes = [P, i32, i32, P, i32, i32]
        L.orc_normalize.argtypes = [P, i32, i32, P]
        L.orc_fill_sample.restype = i32
        L.orc_fill_sample.argtypes = [P, i32, ctypes.c_uint32, i32, i32, i64,
                                      P, P, P, P, P, P, P]
        L.orc_loader_batch.restype = i32
        L.orc_loader_batch.argtypes = [P, P, P, P, P, P, P, i32, P, P, P, P, P, P, i32]
        L.orc_grayscale.argtypes = [P, i32, i32, P]
        L.orc_solarize.argtypes = [P, i32, i32, i32, P]
        L.orc_gaussian_blur.argtypes = [P, i32, i32, P, i32, P]
        L.orc_luma_mean.restype = dbl
        L.orc_luma_mean.argtypes = [P, i32, i32]
        L.orc_adjust.argtypes = [P, i32, i32, i32, dbl, P]
        L.orc_apply_aug_ops.argtypes = [P, i32, i32, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _buf(data: bytes) -> np.ndarray:
    return np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)


class SampleRng:
    """rng.py:34-77 restated over the C oracle."""

    def __init__(self, seed, epoch, index, domain=0):
        self._st = np.array([lib().orc_rng_init(seed & (2**64 - 1), epoch & (2**64 - 1),
                                                index & (2**64 - 1), domain)], np.uint64)

    def next_u64(self):
        return int(lib().orc_rng_next(_p(self._st)))

    def random(self):
        return float(lib().orc_rng_random(_p(self._st)))

    def randint(self, n):
        return int(lib().orc_rng_randint(_p(self._st), n))

    @property
    def state(self):
        return int(self._st[0])


def epoch_permutation(seed, epoch, n):
    out = np.empty(n, np.int64)
    lib().orc_epoch_permutation(seed, epoch, n, _p(out))
    return out


def sample_rrc(rng: SampleRng, w, h, scale=(0.08, 1.0), ratio=(3 / 4, 4 / 3),
               max_attempts=10):
    out = np.zeros(4, np.int32)
    lib().orc_sample_rrc(_p(rng._st), w, h, scale[0], scale[1], ratio[0],
                         ratio[1], max_attempts, _p(out))
    return tuple(int(v) for v in out)


def mask_count(tokens, ratio):
    return int(lib().orc_mask_count(tokens, ratio))


def sample_mask(rng: SampleRng, tokens, k):
    out = np.zeros(max(k, 1), np.int32)
    lib().orc_sample_mask(_p(rng._st), tokens, k, _p(out))
    return out[:k]


def crc32(data: bytes) -> int:
    return int(lib().orc_crc32(_p(_buf(data)), len(data)))


def destuff(raw: bytes, max_restarts=16):
    arr = _buf(raw)
    out = np.zeros(len(raw) + 1, np.uint8)
    rst = np.zeros(max(max_restarts, 1), np.int64)
    nr = np.zeros(1, np.int32)
    end = np.zeros(1, np.int32)
    o = lib().orc_destuff(_p(arr), 0, len(raw), _p(out), _p(rst), max_restarts,
                          _p(nr), _p(end))
    return int(o), int(nr[0]), int(end[0]), out[:o].tobytes(), rst[:min(int(nr[0]), max_restarts)]


def idct_block(coef: np.ndarray, quant: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(coef, np.int32)
    q = np.ascontiguousarray(quant, np.int32)
    out = np.zeros((8, 8), np.uint8)
    lib().orc_idct_block(_p(c), _p(q), _p(out), 8)
    return out


def jpeg_info(data: bytes) -> dict:
    out = np.zeros(12, np.int32)
    err = np.zeros(3, np.int32)
    st = lib().orc_jpeg_info(_p(_buf(data)), len(data), _p(out), _p(err))
    if st:
        raise OracleError(*err)
    keys = ("width", "height", "ncomp", "progressive", "nscans", "ri", "hmax",
            "vmax", "mcus_x", "mcus_y", "scan_start", "scan_end")
    return dict(zip(keys, (int(v) for v in out)))


def decode_crop(data: bytes, rect, full=False):
    """codec.py:448-511. rect = (x, y, w, h). Returns (rgb, (entropy, recon))."""
    if full:
        info = jpeg_info(data)
        x, y, w, h = 0, 0, info["width"], info["height"]
    else:
        x, y, w, h = rect
    out = np.zeros((max(h, 1), max(w, 1), 3), np.uint8)
    stats = np.zeros(2, np.int32)
    err = np.zeros(3, np.int32)
    st = lib().orc_decode_crop(_p(_buf(data)), len(data), x, y, w, h, int(full),
                               _p(out), _p(stats), _p(err))
    if st:
        raise OracleError(*err)
    return out[:h, :w], (int(stats[0]), int(stats[1]))


def decode_full(data: bytes):
    return decode_crop(data, None, full=True)


def dump_coefs(data: bytes, rect):
    """int32 coefficient arrays per component, rows < row_stop (codec.py:483-500)."""
    info = jpeg_info(data)
    cap = 0
    # upper bound: 3 comps x (mcus * 16 blocks) x 64
    cap = 3 * info["mcus_x"] * info["mcus_y"] * 16 * 64 + 64
    out = np.zeros(cap, np.int32)
    dims = np.zeros(6, np.int32)
    err = np.zeros(3, np.int32)
    x, y, w, h = rect
    st = lib().orc_dump_coefs(_p(_buf(data)), len(data), x, y, w, h, _p(out),
                              cap, _p(dims), _p(err))
    if st:
        raise OracleError(*err)
    res, off = [], 0
    for c in range(3):
        bh, bw = int(dims[2 * c]), int(dims[2 * c + 1])
        if bh == 0:
            break
        n = bh * bw * 64
        res.append(out[off:off + n].reshape(bh, bw, 64).copy())
        off += n
    return res


def resize_bilinear(region: np.ndarray, oh: int, ow: int | None = None):
    ow = oh if ow is None else ow
    src = np.ascontiguousarray(region, np.uint8)
    out = np.zeros((oh, ow, 3), np.uint8)
    lib().orc_resize_bilinear(_p(src), src.shape[0], src.shape[1], _p(out), oh, ow)
    return out


def normalize(img: np.ndarray):
    src = np.ascontiguousarray(img, np.uint8)
    out = np.zeros((3, src.shape[0], src.shape[1]), np.float32)
    lib().orc_normalize(_p(src), src.shape[0], src.shape[1], _p(out))
    return out


def _cfg(seed, epoch, res, scale, ratio, mask_grid, mask_k):
    return OrcLoaderCfg(seed & (2**64 - 1), epoch & (2**64 - 1), res, scale[0],
                        scale[1], ratio[0], ratio[1], mask_grid, mask_k)


# ---------------------------------------------------------------------------
# 3-Aug / 3-Aug+ (imgops.py:75-227, pipeline.py:78-101)

SOLARIZE_THRESHOLD = 128          # imgops.py:19
BLUR_SIGMA_RANGE = (0.1, 2.0)     # imgops.py:20
JITTER_STRENGTH = 0.3             # imgops.py:21
AUG_LEVELS = ("simple", "3aug", "3aug+")


class OrcAug(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("ntaps", ctypes.c_int32), ("jitter", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("factors", ctypes.c_double * 3),
                ("wts", ctypes.c_double * 32)]


def blur_weights(sigma: float) -> np.ndarray:
    """gaussian_blur's weights, evaluated with numpy exactly as
    imgops.py:157-160 does (numpy's exp is part of the reference algorithm)."""
    radius = max(1, math.ceil(3.0 * sigma))
    xs = np.arange(-radius, radius + 1, dtype=np.float64)
    wts = np.exp(-(xs * xs) / (2.0 * sigma * sigma))
    wts /= wts.sum()
    return wts


def aug_draws(rng: SampleRng, level: str) -> dict:
    """apply_aug's draws in stream order (pipeline.py:85-101): flip, then
    (3-Aug) op = randint(3) and sigma for the blur, then (3-Aug+) the three
    jitter factors.  `rng` must be positioned after sample_rrc."""
    d = {"flip": int(rng.random() < 0.5), "op": -1, "sigma": None, "factors": None}
    if level != "simple":
        d["op"] = rng.randint(3)
        if d["op"] == 2:
            lo, hi = BLUR_SIGMA_RANGE
            d["sigma"] = lo + (hi - lo) * rng.random()           # rng.py:54-55
    if level == "3aug+":
        s = JITTER_STRENGTH
        d["factors"] = [(1.0 - s) + ((1.0 + s) - (1.0 - s)) * rng.random() for _ in range(3)]
    return d


def orc_aug(d: dict) -> OrcAug:
    a = OrcAug()
    a.op = d["op"]
    if d["op"] == 2:
        w = blur_weights(d["sigma"])
        a.ntaps = len(w)
        for i, v in enumerate(w):
            a.wts[i] = float(v)
    if d["factors"] is not None:
        a.jitter = 1
        for i, v in enumerate(d["factors"]):
            a.factors[i] = v
    return a


def grayscale(img):
    src = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(src)
    lib().orc_grayscale(_p(src), src.shape[0], src.shape[1], _p(out))
    return out


def solarize(img, threshold=SOLARIZE_THRESHOLD):
    src = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(src)
    lib().orc_solarize(_p(src), src.shape[0], src.shape[1], threshold, _p(out))
    return out


def gaussian_blur(img, sigma=None, weights=None):
    src = np.ascontiguousarray(img, np.uint8)
    w = np.ascontiguousarray(blur_weights(sigma) if weights is None else weights, np.float64)
    out = np.empty_like(src)
    lib().orc_gaussian_blur(_p(src), src.shape[0], src.shape[1], _p(w), len(w), _p(out))
    return out


def luma_mean(img):
    src = np.ascontiguousarray(img, np.uint8)
    return float(lib().orc_luma_mean(_p(src), src.shape[0], src.shape[1]))


def _adjust(img, kind, factor):
    src = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(src)
    lib().orc_adjust(_p(src), src.shape[0], src.shape[1], kind, factor, _p(out))
    return out


def adjust_brightness(img, factor):
    return _adjust(img, 0, factor)


def adjust_contrast(img, factor):
    return _adjust(img, 1, factor)


def adjust_saturation(img, factor):
    return _adjust(img, 2, factor)


def apply_aug(rng: SampleRng, img, level: str):
    """pipeline.py:78-101 on an HWC uint8 image."""
    d = aug_draws(rng, level)
    out = np.ascontiguousarray(img[:, ::-1] if d["flip"] else img, np.uint8).copy()
    a = orc_aug(d)
    lib().orc_apply_aug_ops(_p(out), out.shape[0], out.shape[1], ctypes.byref(a))
    return out


def sample_augs(seed, epoch, indices, widths, heights, scale, ratio, level) -> list:
    """Per-sample draws for a batch (rect draws replayed, then aug_draws)."""
    out = []
    for idx in indices:
        r = SampleRng(seed, epoch, int(idx), 0)
        rect = sample_rrc(r, int(widths[idx]), int(heights[idx]), scale, ratio)
        d = aug_draws(r, level)
        d["rect"] = rect
        out.append(d)
    return out


def fill_sample(payload: bytes, crc: int, w: int, h: int, index: int, seed: int,
                epoch: int, res: int, scale=(0.08, 1.0), ratio=(3 / 4, 4 / 3),
                mask_ratio=0.0, patch=16, aug="simple"):
    """pipeline.py:219-235 for one sample -> (pixels f32, u8, mask, rect+flip)."""
    grid = res // patch if mask_ratio > 0 else 0
    k = mask_count(grid * grid, mask_ratio) if grid else 0
    cfg = _cfg(seed, epoch, res, scale, ratio, grid, k)
    pix = np.zeros((3, res, res), np.float32)
    u8 = np.zeros((res, res, 3), np.uint8)
    mask = np.zeros(max(k, 1), np.int32)
    rect = np.zeros(5, np.int32)
    err = np.zeros(3, np.int32)
    a = None
    if aug != "simple":
        r = SampleRng(seed, epoch, index, 0)
        sample_rrc(r, w, h, scale, ratio)
        a = orc_aug(aug_draws(r, aug))
    st = lib().orc_fill_sample(_p(_buf(payload)), len(payload), crc, w, h, index,
                               ctypes.byref(cfg), _p(pix), _p(u8), _p(mask),
                               _p(rect), ctypes.byref(a) if a is not None else None,
                               _p(err))
    if st:
        raise OracleError(*err)
    return pix, u8, (mask[:k] if grid else None), tuple(int(v) for v in rect)


def loader_batch(blob: np.ndarray, records: np.ndarray, indices: np.ndarray,
                 seed: int, epoch: int, res: int, scale=(0.08, 1.0),
                 ratio=(3 / 4, 4 / 3), mask_ratio=0.0, patch=16, keep_uint8=False,
                 nthreads: int | None = None, pixels: np.ndarray | None = None,
                 aug="simple"):
    """A threaded oracle batch over a container mapped as `blob` (uint8)
    with the reference record table `records` (container.py:46-51)."""
    n = len(indices)
    grid = res // patch if mask_ratio > 0 else 0
    k = mask_count(grid * grid, mask_ratio) if grid else 0
    cfg = _cfg(seed, epoch, res, scale, ratio, grid, k)
    if pixels is None:
        pixels = np.empty((n, 3, res, res), np.float32)
    u8 = np.empty((n, res, res, 3), np.uint8) if keep_uint8 else None
    mask = np.empty((n, k), np.int32) if grid else None
    status = np.zeros(n, np.int32)
    offs = np.ascontiguousarray(records["payload_offset"], np.uint64)
    lens = np.ascontiguousarray(records["payload_length"], np.uint32)
    crcs = np.ascontiguousarray(records["checksum"], np.uint32)
    ws = np.ascontiguousarray(records["width"], np.uint16)
    hs = np.ascontiguousarray(records["height"], np.uint16)
    idx = np.ascontiguousarray(indices, np.int64)
    nt = nthreads or os.cpu_count() or 1
    augs = None
    if aug != "simple":
        augs = (OrcAug * max(n, 1))()
        for i, d in enumerate(sample_augs(seed, epoch, idx, ws, hs, scale, ratio, aug)):
            augs[i] = orc_aug(d)
    lib().orc_loader_batch(_p(blob), _p(offs), _p(lens), _p(crcs), _p(ws), _p(hs),
                           _p(idx), n, ctypes.byref(cfg), _p(pixels),
                           _p(u8) if u8 is not None else None,
                           _p(mask) if mask is not None else None, augs, _p(status), nt)
    return pixels, u8, mask, status
