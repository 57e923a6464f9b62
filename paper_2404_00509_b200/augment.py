"""3-Aug / 3-Aug+ stage: host side of the GPU path.

The draws (flip, op, sigma, jitter factors) come from the sample's pipeline
stream in host C++ (essl_aug_draw / essl_aug_batch, pipeline.py:85-101);
the pixel work runs in libessl's k_aug_blur / k_aug_out kernels, either
fused behind the resize (essl_decode_rrc_aug) or standalone on uint8 images
(essl_augment_u8).

Blur weights are the one piece evaluated here: the reference builds them
with numpy's exp (imgops.py:157-160), whose last-ulp results depend on
numpy's SIMD kernels, so the same numpy expression is evaluated on the same
host -- vectorised over all blur samples of a batch, which is element-wise
identical to the per-sample expression (tests/test_host.py pins that).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N

SOLARIZE_THRESHOLD = 128        # imgops.py:19
BLUR_SIGMA_RANGE = (0.1, 2.0)   # imgops.py:20
JITTER_STRENGTH = 0.3           # imgops.py:21

LEVELS = {"simple": N.ESSL_AUG_SIMPLE, "3aug": N.ESSL_AUG_3AUG, "3aug+": N.ESSL_AUG_3AUG_PLUS}


def level_code(level) -> int:
    v = getattr(level, "value", level)
    try:
        return LEVELS[v]
    except KeyError:
        raise ValueError(f"unknown aug level {v!r}") from None


def blur_radius(sigma: float) -> int:
    return max(1, math.ceil(3.0 * sigma))  # imgops.py:156


def blur_weights(sigma: float) -> np.ndarray:
    """gaussian_blur's normalised taps, the reference expression verbatim
    (imgops.py:157-160)."""
    radius = blur_radius(sigma)
    xs = np.arange(-radius, radius + 1, dtype=np.float64)
    wts = np.exp(-(xs * xs) / (2.0 * sigma * sigma))
    wts /= wts.sum()
    return wts


def fill_weights(aug: np.ndarray) -> np.ndarray:
    """Write the blur taps of every blur entry of an N.aug_dtype() array
    (in place), grouped by radius so each group is one numpy expression."""
    blur = np.nonzero(aug["op"] == N.ESSL_AUG_OP_BLUR)[0]
    if blur.size == 0:
        return aug
    radii = aug["radius"][blur]
    for r in np.unique(radii):
        r = int(r)
        if not 1 <= r <= N.ESSL_AUG_MAX_RADIUS:
            raise ValueError(f"blur radius {r} out of range")
        rows = blur[radii == r]
        sig = aug["sigma"][rows]
        xs = np.arange(-r, r + 1, dtype=np.float64)
        w = np.exp(-(xs * xs)[None, :] / (2.0 * sig * sig)[:, None])
        w /= w.sum(axis=1, keepdims=True)
        aug["weights"][rows, :2 * r + 1] = w
        aug["weights"][rows, 2 * r + 1:] = 0.0
    return aug


def new_aug(n: int) -> np.ndarray:
    a = np.zeros(n, N.aug_dtype())
    a["op"] = N.ESSL_AUG_OP_NONE
    a["threshold"] = SOLARIZE_THRESHOLD
    return a


def draw(state, level) -> tuple[int, np.ndarray]:
    """apply_aug's draws from a ctypes uint64 stream state (advanced in
    place): returns (flip, one-entry aug array with weights filled)."""
    import ctypes
    a = new_aug(1)
    flip = ctypes.c_int32(0)
    N.check(N.lib().essl_aug_draw(ctypes.byref(state), level_code(level), ctypes.byref(flip),
                                  N.ptr(a)), "essl_aug_draw")
    return int(flip.value), fill_weights(a)


def any_work(aug: np.ndarray | None) -> bool:
    return aug is not None and bool(((aug["op"] != N.ESSL_AUG_OP_NONE) | (aug["jitter"] != 0)).any())


# ---- standalone ops on uint8 HWC images (imgops.py:75-227) ------------------

def _run(img, aug: np.ndarray, device=None):
    import torch
    from .engine import default_engine
    eng = default_engine(device)
    was_np = not isinstance(img, torch.Tensor)
    src = (torch.from_numpy(np.ascontiguousarray(img, np.uint8)) if was_np else img)
    src = src.to(eng.device).contiguous()
    if src.ndim != 3 or src.shape[2] != 3:
        raise ValueError(f"expected (h, w, 3) uint8 image, got {tuple(src.shape)}")
    dst = torch.empty_like(src)
    eng.augment_u8(src[None], aug, dst[None])
    return dst.cpu().numpy() if was_np else dst


def grayscale(img, device=None):
    a = new_aug(1)
    a["op"] = N.ESSL_AUG_OP_GRAY
    return _run(img, a, device)


def solarize(img, threshold: int = SOLARIZE_THRESHOLD, device=None):
    a = new_aug(1)
    a["op"] = N.ESSL_AUG_OP_SOLARIZE
    a["threshold"] = threshold
    return _run(img, a, device)


def gaussian_blur(img, sigma: float, device=None):
    a = new_aug(1)
    a["op"] = N.ESSL_AUG_OP_BLUR
    a["sigma"] = sigma
    a["radius"] = blur_radius(sigma)
    return _run(img, fill_weights(a), device)


def color_jitter(img, brightness: float, contrast: float, saturation: float, device=None):
    """adjust_brightness -> adjust_contrast -> adjust_saturation
    (pipeline.py:97-101) in one pass."""
    a = new_aug(1)
    a["jitter"] = 1
    a["factors"][0] = (brightness, contrast, saturation)
    return _run(img, a, device)
