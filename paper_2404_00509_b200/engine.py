"""Device engine: one libessl context per (device, consumer), torch for device
memory and streams, ctypes for the C ABI (include/essl.h).

Every GPU entry point of the package goes through an Engine; the library is
required (no CPU fallback -- _native.lib() raises NativeUnavailable).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N
from .errors import status_error


def _torch():
    import torch
    return torch


class Engine:
    """A libessl context bound to one CUDA device.

    Capacities (batch, max side, max payload) grow on demand by recreating
    the context; steady-state loader use never reallocates.
    """

    def __init__(self, device=None, max_batch: int = 16, max_side: int = 512,
                 max_payload: int = 1 << 18):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required (libessl has no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._ctx = ctypes.c_void_p()
        self._caps = (0, 0, 0)
        self._options = {}
        self._ensure(max_batch, max_side, max_payload)
        self._sample_dtype, self._result_dtype = N._np_dtypes()

    # ---- context management ------------------------------------------------
    def _ensure(self, batch: int, side: int, payload: int) -> None:
        b, s, p = self._caps
        if batch <= b and side <= s and payload <= p:
            return
        nb, ns, np_ = max(batch, b), max(side, s), max(payload, p)
        self.close()
        torch = _torch()
        with torch.cuda.device(self.device):
            torch.cuda.init()
            N.check(N.lib().essl_ctx_create(self.device.index, nb, ns, np_, 0,
                                            ctypes.byref(self._ctx)), "essl_ctx_create")
        self._caps = (nb, ns, np_)
        for k, v in self._options.items():
            N.check(N.lib().essl_ctx_set_option(self._ctx, k, v), "essl_ctx_set_option")

    def set_option(self, option: int, value: int) -> None:
        self._options[option] = int(value)
        N.check(N.lib().essl_ctx_set_option(self._ctx, option, int(value)), "essl_ctx_set_option")

    def close(self) -> None:
        if self._ctx:
            N.lib().essl_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(N.lib().essl_ctx_launch_count(self._ctx)) if self._ctx else 0

    def profile_read(self) -> dict:
        """{kernel: (total_ms, launches)} since the last read (ESSL_OPT_PROFILE)."""
        ms = np.zeros(len(N.KERNELS), np.float64)
        cnt = np.zeros(len(N.KERNELS), np.int64)
        N.check(N.lib().essl_ctx_profile_read(self._ctx, N.ptr(ms), N.ptr(cnt)),
                "essl_ctx_profile_read")
        out = {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(N.KERNELS) if cnt[i]}
        parts = [out[k] for k in ("prep", "entropy", "idct") if k in out]
        if parts:  # the whole decode stage: k_prep + k_entropy + k_idct
            out["decode"] = (sum(p[0] for p in parts), max(p[1] for p in parts))
        return out

    def profile_timeline(self, max_records: int = 1 << 16) -> list:
        """[(kernel, start_ms, end_ms)] after the last essl_profile_mark
        (ESSL_OPT_PROFILE on; call before profile_read, which clears)."""
        kid = np.zeros(max_records, np.int32)
        t0 = np.zeros(max_records, np.float64)
        t1 = np.zeros(max_records, np.float64)
        n = N.lib().essl_ctx_profile_timeline(self._ctx, N.ptr(kid), N.ptr(t0), N.ptr(t1), max_records)
        N.check(min(n, 0), "essl_ctx_profile_timeline")
        return [(N.KERNELS[kid[i]], float(t0[i]), float(t1[i])) for i in range(n)]

    def stream(self):
        return _torch().cuda.current_stream(self.device)

    def _st(self, stream=None):
        s = stream if stream is not None else self.stream()
        return ctypes.c_void_p(s.cuda_stream)

    # ---- descriptors ---------------------------------------------------------
    def samples(self, n: int) -> np.ndarray:
        return np.zeros(n, self._sample_dtype)

    # ---- hot path ------------------------------------------------------------
    def stage(self, slot: int, ptrs: np.ndarray, lens: np.ndarray, samples: np.ndarray,
              nthreads: int = 8, stream=None):
        """Gather host payloads (addresses in ``ptrs``) into pinned memory and
        copy them to the device; fills samples['offset'/'length']."""
        n = len(samples)
        self._ensure(n, 0, int(lens.max()) if n else 0)
        blob = ctypes.c_void_p()
        p = np.ascontiguousarray(ptrs, np.uint64)
        ln = np.ascontiguousarray(lens, np.uint32)
        N.check(N.lib().essl_stage(self._ctx, slot, N.ptr(p), N.ptr(ln), n, N.ptr(samples),
                                   nthreads, self._st(stream), ctypes.byref(blob)), "essl_stage")
        return blob.value

    def stage_pinned(self, slot: int, host_base: int, offsets: np.ndarray, lens: np.ndarray,
                     samples: np.ndarray, stream=None):
        """Gather payloads of a page-locked container (host_base + offsets)
        host->device with one batched copy; fills samples['offset'/'length']."""
        n = len(samples)
        self._ensure(n, 0, int(lens.max()) if n else 0)
        blob = ctypes.c_void_p()
        o = np.ascontiguousarray(offsets, np.uint64)
        ln = np.ascontiguousarray(lens, np.uint32)
        N.check(N.lib().essl_stage_pinned(self._ctx, slot, ctypes.c_void_p(host_base), N.ptr(o), N.ptr(ln),
                                          n, N.ptr(samples), self._st(stream), ctypes.byref(blob)),
                "essl_stage_pinned")
        return blob.value

    def decode_rrc(self, blob_ptr: int, samples: np.ndarray, res: int, out_kind: int,
                   out=None, out_u8=None, results=None, stream=None, max_side: int = 0,
                   aug: np.ndarray | None = None, out_stride: int = 0, vis=None):
        """Decode + RRC resize + flip (+ 3-Aug stage when ``aug``, an
        N.aug_dtype() array with blur weights filled) + normalize.  ``vis``:
        (patch, ids_restore, tokens) for the fused visible-token output."""
        n = len(samples)
        self._ensure(n, max_side, int(samples["length"].max()) if n else 0)
        patch, restore, tokens = vis if vis is not None else (0, None, None)
        n_keep = int(tokens.shape[1]) if tokens is not None else 0
        N.check(N.lib().essl_decode_rrc_visible(
            self._ctx, ctypes.c_void_p(blob_ptr), N.ptr(samples), N.ptr(aug), n, res, out_kind,
            N.ptr(out), out_stride, N.ptr(out_u8), patch if tokens is not None else 0,
            N.ptr(restore if tokens is not None else None), n_keep, N.ptr(tokens), N.ptr(results),
            self._st(stream)), "essl_decode_rrc")

    def augment_u8(self, src, aug: np.ndarray, dst, stream=None):
        """apply_aug's pixel stage on device uint8 [n,h,w,3] images."""
        n, h, w = int(src.shape[0]), int(src.shape[1]), int(src.shape[2])
        self._ensure(n, max(h, w), 0)
        N.check(N.lib().essl_augment_u8(self._ctx, N.ptr(src), n, h, w, N.ptr(aug), N.ptr(dst),
                                        self._st(stream)), "essl_augment_u8")

    def decode_crop_u8(self, blob_ptr: int, samples: np.ndarray, out, offsets: np.ndarray,
                       results=None, stream=None, max_side: int = 0):
        n = len(samples)
        self._ensure(n, max_side, int(samples["length"].max()) if n else 0)
        off = np.ascontiguousarray(offsets, np.uint64)
        N.check(N.lib().essl_decode_crop_u8(self._ctx, ctypes.c_void_p(blob_ptr), N.ptr(samples),
                                            n, N.ptr(out), N.ptr(off), N.ptr(results),
                                            self._st(stream)), "essl_decode_crop_u8")

    def dump_coefs(self, blob_ptr: int, samples: np.ndarray, out, offsets: np.ndarray,
                   cap: int, results=None, stream=None, max_side: int = 0) -> np.ndarray:
        n = len(samples)
        self._ensure(n, max_side, int(samples["length"].max()) if n else 0)
        geo = np.zeros(12 * n, np.int32)
        off = np.ascontiguousarray(offsets, np.uint64)
        N.check(N.lib().essl_dump_coefs(self._ctx, ctypes.c_void_p(blob_ptr), N.ptr(samples), n,
                                        N.ptr(out), N.ptr(off), cap, N.ptr(geo), N.ptr(results),
                                        self._st(stream)), "essl_dump_coefs")
        return geo.reshape(n, 3, 4)

    def mask(self, seed: int, epoch: int, index_dev, tokens: int, k: int, mask=None, keep=None,
             restore=None, stream=None):
        n = int(index_dev.shape[0])
        N.check(N.lib().essl_mask(self._ctx, seed & (2**64 - 1), epoch & (2**64 - 1),
                                  N.ptr(index_dev), n, tokens, k, N.ptr(mask), N.ptr(keep),
                                  N.ptr(restore), self._st(stream)), "essl_mask")

    def gather_visible(self, pixels_bf16, res: int, patch: int, ids_keep, tokens_out,
                       stream=None):
        n, n_keep = int(ids_keep.shape[0]), int(ids_keep.shape[1])
        N.check(N.lib().essl_gather_visible(self._ctx, N.ptr(pixels_bf16), n, res, patch,
                                            N.ptr(ids_keep), n_keep, N.ptr(tokens_out),
                                            self._st(stream)), "essl_gather_visible")

    # ---- results ---------------------------------------------------------------
    def new_results(self, n: int):
        torch = _torch()
        return torch.empty((n, ctypes.sizeof(N.EsslResult) // 4), dtype=torch.int32,
                           device=self.device)

    def raise_for(self, results_host: np.ndarray, samples: np.ndarray,
                  sample_ids=None) -> None:
        """Raise the reference exception for the first failing image."""
        st = results_host[:, 0]
        bad = np.nonzero(st != 0)[0]
        if bad.size == 0:
            return
        i = int(bad[0])
        r = results_host[i]
        s = samples[i]
        raise status_error(int(r[0]), int(r[1]), int(r[2]),
                           sample=None if sample_ids is None else int(sample_ids[i]),
                           rect=(int(s["x"]), int(s["y"]), int(s["w"]), int(s["h"])),
                           dims=(int(r[5]), int(r[6])))


_engines: dict = {}
_lock = threading.Lock()


def default_engine(device=None) -> Engine:
    """Per-thread, per-device engine for the functional API."""
    torch = _torch()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (threading.get_ident(), dev.index)
    with _lock:
        eng = _engines.get(key)
        if eng is None:
            eng = _engines[key] = Engine(dev)
    return eng
