"""Standalone pixel ops on the GPU (mirror of cropload/imgops.py:16-21, 63-72,
75-227, 243-257).  Inputs may be numpy arrays (copied to the device and
back) or CUDA tensors (stay on the device)."""

from __future__ import annotations

import numpy as np

from . import _native as N
from .engine import default_engine

IMAGENET_MEAN = np.array([0.485, 0.456, 0.406], np.float32)
IMAGENET_STD = np.array([0.229, 0.224, 0.225], np.float32)

from .augment import (BLUR_SIGMA_RANGE, JITTER_STRENGTH, SOLARIZE_THRESHOLD,  # noqa: E402,F401
                      gaussian_blur, grayscale, solarize)
from .augment import color_jitter as _color_jitter  # noqa: E402


def adjust_brightness(img, factor: float):
    """imgops.py:213-216 (factor 1.0 leaves the other two stages identity)."""
    return _color_jitter(img, factor, 1.0, 1.0)


def adjust_contrast(img, factor: float):
    """imgops.py:219-222: blend with the image's mean BT.601 luma."""
    return _color_jitter(img, 1.0, factor, 1.0)


def adjust_saturation(img, factor: float):
    """imgops.py:225-227: blend with the per-pixel grayscale."""
    return _color_jitter(img, 1.0, 1.0, factor)


def _to_dev(a, eng):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(eng.device).contiguous(), False
    a = np.ascontiguousarray(a, np.uint8)
    if not a.flags.writeable:  # (read-only views, e.g. Pillow buffers: copy before wrapping)
        a = a.copy()
    return torch.from_numpy(a).to(eng.device), True


def resize_bilinear(region, out_h: int, out_w: int | None = None, flip: bool = False,
                    device=None):
    """Half-pixel bilinear resize, float64, round-half-up (imgops.py:24-72);
    ``flip`` folds hflip (imgops.py:256) into the output index."""
    import torch
    if out_w is None:
        out_w = out_h
    if region.ndim != 3 or region.shape[2] != 3 or region.shape[0] < 1 or region.shape[1] < 1:
        raise ValueError(f"expected nonempty (h, w, 3) region, got {tuple(region.shape)}")
    eng = default_engine(device)
    src, was_np = _to_dev(region, eng)
    out = torch.empty((out_h, out_w, 3), dtype=torch.uint8, device=eng.device)
    N.check(N.lib().essl_resize_u8(N.ptr(src), src.shape[0], src.shape[1], N.ptr(out), out_h,
                                   out_w, int(flip), eng._st()), "essl_resize_u8")
    return out.cpu().numpy() if was_np else out


def normalize(img, out=None, device=None):
    """HWC uint8 -> CHW float32 ImageNet normalisation (imgops.py:231-248)."""
    import torch
    eng = default_engine(device)
    src, was_np = _to_dev(img, eng)
    h, w = src.shape[0], src.shape[1]
    dst = torch.empty((3, h, w), dtype=torch.float32, device=eng.device)
    N.check(N.lib().essl_normalize_u8(N.ptr(src), h, w, N.ptr(dst), eng._st()),
            "essl_normalize_u8")
    if was_np:
        res = dst.cpu().numpy()
        if out is not None:
            out[...] = res
            return out
        return res
    if out is not None:
        out.copy_(dst)
        return out
    return dst


def denormalize(chw):
    """Inverse of normalize, back to [0, 1] floats (imgops.py:251-253)."""
    return chw * IMAGENET_STD[:, None, None] + IMAGENET_MEAN[:, None, None]


def hflip(img):
    """imgops.py:256-257."""
    import torch
    if isinstance(img, torch.Tensor):
        return torch.flip(img, dims=[1]).contiguous()
    return np.ascontiguousarray(img[:, ::-1])
