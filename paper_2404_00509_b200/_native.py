"""ctypes binding of libessl (include/essl.h).

The library is built in-tree by ``paper_2404_00509_b200.build`` (nvcc,
sm_100a).  There is no CPU fallback: if the library is missing, every GPU
entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

# ESSL_LIB: an alternative build of the library (A/B experiments, tools/ab.py)
LIB_PATH = Path(os.environ.get("ESSL_LIB") or Path(__file__).resolve().parent / "_lib" / "libessl.so")

ESSL_OK = 0
ESSL_OUT_BF16_NCHW, ESSL_OUT_F32_NCHW, ESSL_OUT_NONE = 0, 1, 2
ESSL_DECODE_SPECULATIVE, ESSL_DECODE_SERIAL = 0, 1
ESSL_OPT_DECODE_MODE, ESSL_OPT_SEQ_BITS, ESSL_OPT_CHECKPOINT_BITS, ESSL_OPT_PROFILE = 1, 2, 3, 4
ESSL_OPT_WARMUP_BITS = 5
ESSL_OPT_STAGE_BYTES = 6
ESSL_OPT_GATHER_CTAS = 7
ESSL_OPT_GATHER_TMA = 8
ESSL_OPT_DEBUG_LANES = 9
ESSL_OPT_TRACE = 10
ESSL_OPT_RESIZE_COLS = 11
ESSL_OPT_RESIZE_BAND = 12
ESSL_OPT_EARLY_EXIT = 13
ESSL_OPT_PROFILE_KERNELS = 14
ESSL_K_ENTROPY = 7
KERNELS = ("decode", "resize", "crop_u8", "mask", "gather", "dump_coefs", "prep", "entropy", "idct",
           "stage", "aug")
ESSL_AUG_SIMPLE, ESSL_AUG_3AUG, ESSL_AUG_3AUG_PLUS = 0, 1, 2
ESSL_AUG_OP_NONE, ESSL_AUG_OP_GRAY, ESSL_AUG_OP_SOLARIZE, ESSL_AUG_OP_BLUR = -1, 0, 1, 2
ESSL_AUG_MAX_RADIUS = 12

# Every symbol include/essl.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "essl_ctx_create", "essl_ctx_destroy", "essl_ctx_set_option", "essl_ctx_launch_count",
    "essl_ctx_profile_read", "essl_profile_mark", "essl_ctx_profile_timeline", "essl_debug_stats",
    "essl_last_error", "essl_version", "essl_stage", "essl_stage_pinned", "essl_host_register",
    "essl_host_unregister", "essl_host_device_ptr", "essl_decode_rrc", "essl_decode_crop_u8",
    "essl_dump_coefs", "essl_mask", "essl_mask_from_states", "essl_gather_visible", "essl_resize_u8",
    "essl_normalize_u8", "essl_rng_init", "essl_rng_next", "essl_rng_random",
    "essl_rng_randint", "essl_epoch_permutation", "essl_sample_rrc", "essl_rrc_batch",
    "essl_mask_count", "essl_encode_jpeg", "essl_synth_image", "essl_decode_rrc_aug",
    "essl_augment_u8", "essl_aug_draw", "essl_aug_batch", "essl_debug_lanes",
    "essl_trace_read", "essl_memcpy_async", "essl_option_default",
    "essl_decode_rrc_visible", "essl_dataset_create", "essl_dataset_destroy", "essl_batch_enqueue", "essl_abi_sizes",
    "essl_check_read",
)


class NativeUnavailable(RuntimeError):
    pass


class EsslSample(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_uint64), ("length", ctypes.c_uint32),
                ("crc32", ctypes.c_uint32), ("x", ctypes.c_int32), ("y", ctypes.c_int32),
                ("w", ctypes.c_int32), ("h", ctypes.c_int32), ("flip", ctypes.c_int32),
                ("check_crc", ctypes.c_int32)]


class EsslResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("reason", ctypes.c_int32),
                ("offset", ctypes.c_int32), ("mcus_entropy_decoded", ctypes.c_int32),
                ("mcus_reconstructed", ctypes.c_int32), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32), ("ncomp", ctypes.c_int32)]


class EsslAug(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("radius", ctypes.c_int32), ("jitter", ctypes.c_int32),
                ("threshold", ctypes.c_int32), ("sigma", ctypes.c_double),
                ("factors", ctypes.c_double * 3),
                ("weights", ctypes.c_double * (2 * ESSL_AUG_MAX_RADIUS + 1)),
                ("reserved", ctypes.c_double)]


class EsslBatchCfg(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("epoch", ctypes.c_uint64),
                ("scale", ctypes.c_double * 2), ("ratio", ctypes.c_double * 2),
                ("res", ctypes.c_int32), ("out_kind", ctypes.c_int32), ("check_crc", ctypes.c_int32),
                ("tokens", ctypes.c_int32), ("masked", ctypes.c_int32), ("patch", ctypes.c_int32)]


class EsslBatchIo(ctypes.Structure):
    _fields_ = [("blob", ctypes.c_void_p), ("pinned_base", ctypes.c_void_p),
                ("stage_slot", ctypes.c_int32), ("stage_chain", ctypes.c_int32), ("aug", ctypes.c_void_p),
                ("pixels", ctypes.c_void_p), ("pixel_stride", ctypes.c_int64),
                ("u8", ctypes.c_void_p), ("index_label", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("ids_keep", ctypes.c_void_p), ("ids_restore", ctypes.c_void_p),
                ("tokens", ctypes.c_void_p), ("results", ctypes.c_void_p),
                ("results_host", ctypes.c_void_p), ("wait_stream", ctypes.c_void_p)]


SAMPLE_NP_DTYPE = None  # filled lazily (numpy view of EsslSample arrays)
RESULT_NP_DTYPE = None
AUG_NP_DTYPE = None

_lib = None


def aug_dtype():
    """numpy view of EsslAug arrays."""
    global AUG_NP_DTYPE
    import numpy as np
    if AUG_NP_DTYPE is None:
        AUG_NP_DTYPE = np.dtype([("op", "<i4"), ("radius", "<i4"), ("jitter", "<i4"),
                                 ("threshold", "<i4"), ("sigma", "<f8"), ("factors", "<f8", 3),
                                 ("weights", "<f8", 2 * ESSL_AUG_MAX_RADIUS + 1),
                                 ("reserved", "<f8")])
        assert AUG_NP_DTYPE.itemsize == ctypes.sizeof(EsslAug)
    return AUG_NP_DTYPE


def _np_dtypes():
    global SAMPLE_NP_DTYPE, RESULT_NP_DTYPE
    import numpy as np
    if SAMPLE_NP_DTYPE is None:
        SAMPLE_NP_DTYPE = np.dtype([("offset", "<u8"), ("length", "<u4"), ("crc32", "<u4"),
                                    ("x", "<i4"), ("y", "<i4"), ("w", "<i4"), ("h", "<i4"),
                                    ("flip", "<i4"), ("check_crc", "<i4")])
        assert SAMPLE_NP_DTYPE.itemsize == ctypes.sizeof(EsslSample)
        RESULT_NP_DTYPE = np.dtype([(n, "<i4") for n, _ in EsslResult._fields_])
        assert RESULT_NP_DTYPE.itemsize == ctypes.sizeof(EsslResult)
    return SAMPLE_NP_DTYPE, RESULT_NP_DTYPE


def lib():
    """Load libessl.so (raises NativeUnavailable if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} not built; run `python -m paper_2404_00509_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.c_void_p
    i32, i64, u64, dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "essl_ctx_create": (i32, [i32, i32, i32, i32, i32, P]),
        "essl_ctx_destroy": (i32, [P]),
        "essl_ctx_set_option": (i32, [P, i32, i64]),
        "essl_option_default": (i32, [i32, P]),
        "essl_ctx_launch_count": (i64, [P]),
        "essl_ctx_profile_read": (i32, [P, P, P]),
        "essl_profile_mark": (i32, [P]),
        "essl_ctx_profile_timeline": (i32, [P, P, P, P, i32]),
        "essl_debug_stats": (i32, [P, P, i32]),
        "essl_debug_lanes": (i32, [P, P, i32]),
        "essl_trace_read": (i32, [P, P, i32]),
        "essl_last_error": (ctypes.c_char_p, []),
        "essl_memcpy_async": (i32, [P, P, u64, P]),
        "essl_version": (ctypes.c_char_p, []),
        "essl_stage": (i32, [P, i32, P, P, i32, P, i32, P, P]),
        "essl_stage_pinned": (i32, [P, i32, P, P, P, i32, P, P, P]),
        "essl_host_register": (i32, [P, ctypes.c_uint64, i32]),
        "essl_host_unregister": (i32, [P]),
        "essl_host_device_ptr": (i32, [P, P]),
        "essl_decode_rrc": (i32, [P, P, P, i32, i32, i32, P, i64, P, P, P]),
        "essl_decode_crop_u8": (i32, [P, P, P, i32, P, P, P, P]),
        "essl_dump_coefs": (i32, [P, P, P, i32, P, P, i64, P, P, P]),
        "essl_mask": (i32, [P, u64, u64, P, i32, i32, i32, P, P, P, P]),
        "essl_mask_from_states": (i32, [P, P, i32, i32, i32, P, P, P, P]),
        "essl_gather_visible": (i32, [P, P, i32, i32, i32, P, i32, P, P]),
        "essl_resize_u8": (i32, [P, i32, i32, P, i32, i32, i32, P]),
        "essl_normalize_u8": (i32, [P, i32, i32, P, P]),
        "essl_rng_init": (u64, [u64, u64, u64, u64]),
        "essl_rng_next": (u64, [P]),
        "essl_rng_random": (dbl, [P]),
        "essl_rng_randint": (i64, [P, i64]),
        "essl_epoch_permutation": (i32, [u64, u64, i64, P]),
        "essl_sample_rrc": (i32, [P, i64, i64, dbl, dbl, dbl, dbl, i32, P]),
        "essl_rrc_batch": (i32, [u64, u64, P, i32, P, P, dbl, dbl, dbl, dbl, P]),
        "essl_mask_count": (i32, [i32, dbl]),
        "essl_encode_jpeg": (i64, [P, i32, i32, i32, i32, P, i64]),
        "essl_synth_image": (i32, [u64, i32, i32, P]),
        "essl_decode_rrc_aug": (i32, [P, P, P, P, i32, i32, i32, P, i64, P, P, P]),
        "essl_augment_u8": (i32, [P, P, i32, i32, i32, P, P, P]),
        "essl_dataset_create": (i32, [i64, P, P, P, P, P, P, P]),
        "essl_dataset_destroy": (i32, [P]),
        "essl_batch_enqueue": (i32, [P, P, P, P, i32, P, P]),
        "essl_abi_sizes": (i32, [P, i32]),
        "essl_check_read": (i32, [P, i32, i32]),
        "essl_decode_rrc_visible": (i32, [P, P, P, P, i32, i32, i32, P, i64, P, i32, P, i32, P,
                                          P, P]),
        "essl_aug_draw": (i32, [P, i32, P, P]),
        "essl_aug_batch": (i32, [u64, u64, P, i32, P, P, dbl, dbl, dbl, dbl, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def option_default(option: int) -> int:
    """The value a new libessl context starts with for ESSL_OPT_* `option`."""
    v = ctypes.c_int64()
    check(lib().essl_option_default(option, ctypes.byref(v)), "essl_option_default")
    return int(v.value)


def check(rc: int, what: str = "libessl") -> None:
    if rc != ESSL_OK:
        msg = lib().essl_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def ptr(a) -> ctypes.c_void_p | None:
    """Raw pointer of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)
