"""GPU drop-in for the reference sample pipeline (cropload/pipeline.py).

Same API surface -- ``RrcConfig``, ``sample_rrc``, ``apply_aug``,
``ImageBatch``, ``LoaderConfig`` (same JSON keys), ``Loader`` with
``epoch(e)`` / ``batches_per_epoch`` / context manager -- and the same
determinism contract: every sample is a pure function of (bytes, config,
seed, epoch, index), so batch content matches the reference bit for bit
(float32 mode) no matter how work is scheduled.

Per batch (pipeline.py:219-267):
  host C++   : epoch permutation, DDP shard, RRC rect + flip (+ 3-Aug draws)
               per sample (glibc libm, bit-exact with CPython), descriptor
               table; blur taps via numpy (the reference's own expression)
  GPU        : CRC32 -> parse -> destuff -> speculative Huffman decode of the
               crop's MCU rows -> IDCT of crop MCUs -> colour + bilinear +
               flip [-> 3-Aug/3-Aug+ stage] -> normalize -> bf16/f32 NCHW
               (+ uint8 NHWC) ;
               MAE mask + ids_keep/ids_restore
Compressed bytes are either HBM-resident (the container uploaded once) or
staged per batch through a pinned double buffer.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
from collections import deque
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .container import ContainerHandle, open_container
from .errors import ConfigError, CorruptionError
from .jpeg import CropRect
from .masking import MaskSpec
from .rng import SampleRng, epoch_permutation, shard, shard_len
from .schedule import AugLevel


@dataclass(frozen=True)
class RrcConfig:
    """RandomResizedCrop distribution (pipeline.py:31-48)."""

    scale: tuple = (0.08, 1.0)
    ratio: tuple = (3.0 / 4.0, 4.0 / 3.0)
    out_size: int = 224
    max_attempts: int = 10

    def __post_init__(self):
        if not 0.0 < self.scale[0] <= self.scale[1] <= 1.0:
            raise ConfigError(f"scale bounds must satisfy 0 < lo <= hi <= 1: {self.scale}")
        if not 0.0 < self.ratio[0] <= self.ratio[1]:
            raise ConfigError(f"ratio bounds must be positive and ordered: {self.ratio}")
        if self.out_size < 16:
            raise ConfigError(f"output size must be >= 16: {self.out_size}")
        if self.max_attempts < 1:
            raise ConfigError("max_attempts must be >= 1")


def sample_rrc(rng: SampleRng, src_w: int, src_h: int, cfg: RrcConfig) -> CropRect:
    """Crop window draw (pipeline.py:51-75), native host C++ (glibc libm)."""
    import ctypes
    out = np.zeros(4, np.int32)
    N.check(N.lib().essl_sample_rrc(ctypes.byref(rng._state), src_w, src_h, cfg.scale[0],
                                    cfg.scale[1], cfg.ratio[0], cfg.ratio[1], cfg.max_attempts,
                                    N.ptr(out)), "essl_sample_rrc")
    return CropRect(int(out[0]), int(out[1]), int(out[2]), int(out[3]))


def apply_aug(rng: SampleRng, img, level: AugLevel):
    """Simple / 3-aug / 3-aug+ augmentation, all draws from ``rng``
    (pipeline.py:78-101): flip at p=0.5, then (3-aug) one of grayscale,
    solarize, gaussian blur, then (3-aug+) brightness / contrast /
    saturation jitter.  Draws in host C++, pixels on the GPU (k_aug_*)."""
    from . import augment
    from .imgops import hflip
    flip, a = augment.draw(rng._state, level)
    if flip:
        img = hflip(img)
    if augment.any_work(a):
        img = augment._run(img, a)
    return img


@dataclass
class ImageBatch:
    """One assembled batch (pipeline.py:105-117); tensors live on the GPU.

    pixels: [b,3,h,h] float32 (reference dtype) or bfloat16; labels/indices
    int64 [b]; mask int32 [b,k] sorted masked ids; uint8 [b,h,h,3] view;
    ids_keep int64 [b,N-k]; ids_restore int64 [b,N]; visible bf16
    [b,N-k,p*p*3] (optional)."""

    pixels: object
    labels: object
    indices: object
    epoch: int
    mask: object = None
    uint8: object = None
    ids_keep: object = None
    ids_restore: object = None
    # MAE visible tokens (LoaderConfig.visible): bf16 [b, N-k, patch*patch*3],
    # patchify 'nchpwq->nhwpqc' of pixels gathered at ids_keep
    visible: object = None

    def __len__(self) -> int:
        return int(self.pixels.shape[0])


_GPU_KEYS = ("reuse_outputs", "device", "out_dtype", "rank", "world_size", "resident", "prefetch",
             "streams", "staging", "shard_mode", "visible", "group", "fill_chain")


@dataclass
class LoaderConfig:
    """pipeline.py:120-170 plus GPU-only keys (device, out_dtype, rank,
    world_size, resident, prefetch)."""

    data: str
    batch_size: int = 256
    workers: int = 0
    seed: int = 0
    res: int = 224
    scale: tuple = (0.08, 1.0)
    ratio: tuple = (3.0 / 4.0, 4.0 / 3.0)
    aug: str = "simple"
    mask_ratio: float = 0.0
    patch: int = 16
    keep_uint8: bool = False
    # GPU extensions
    device: str | None = None
    out_dtype: str = "float32"
    rank: int = 0
    world_size: int = 1
    resident: bool = True
    # host container (resident=False) payload path: "gather" = a few-CTA
    # kernel reads the page-locked container over the bus; "copy" = host
    # threads gather into a pinned ring, one copy-engine transfer per batch
    staging: str = "gather"
    prefetch: int = 2
    streams: int = 2
    # Reuse a ring of output buffers (a batch's views stay valid while fewer
    # than `prefetch + 2` later batches have been issued -- the reference
    # bindings' "valid until the next step" contract) instead of
    # allocating every batch.
    reuse_outputs: bool = False
    # DDP partition of each epoch's permutation (rng.shard): "pad" (equal
    # shards, DistributedSampler default), "drop" or "stride" (perm[r::world])
    shard_mode: str = "pad"
    # emit ImageBatch.visible: the MAE encoder's visible tokens, written by the
    # resize kernel itself (needs mask_ratio > 0)
    visible: bool = False
    # the iterators (epoch / epochs) decode up to `group` consecutive batches
    # of one epoch in one launch set (the same batches, fewer and larger
    # launches); enqueue() is always one batch
    group: int = 1
    # host-staged containers: while the iterators fill the pipeline, each
    # batch's bus gather waits for the previous one and runs on this many
    # CTAs (the oldest batch's payloads arrive first); 0 (default since the
    # gather's 4 KB stages): all concurrent
    fill_chain: int = 0

    _KEYS = ("data", "batch_size", "workers", "seed", "res", "scale", "ratio", "aug",
             "mask_ratio", "patch", "keep_uint8") + _GPU_KEYS

    @classmethod
    def from_document(cls, doc) -> "LoaderConfig":
        if isinstance(doc, Path) or (isinstance(doc, str) and not doc.lstrip().startswith("{")):
            doc = Path(doc).read_text()
        if isinstance(doc, str):
            doc = json.loads(doc)
        if not isinstance(doc, dict):
            raise ConfigError("loader config must be a JSON object")
        unknown = set(doc) - set(cls._KEYS)
        if unknown:
            raise ConfigError(f"unknown loader config keys: {sorted(unknown)}")
        if "data" not in doc:
            raise ConfigError("loader config missing required key: data")
        kw = dict(doc)
        for key in ("scale", "ratio"):
            if key in kw:
                v = kw[key]
                if not (isinstance(v, (list, tuple)) and len(v) == 2):
                    raise ConfigError(f"{key} must be a [lo, hi] pair")
                kw[key] = (float(v[0]), float(v[1]))
        return cls(**kw)

    def validate(self) -> None:
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if self.aug not in tuple(a.value for a in AugLevel):
            raise ConfigError(f"aug must be one of {[a.value for a in AugLevel]}, got {self.aug!r}")
        if not 0.0 <= self.mask_ratio <= 1.0:
            raise ConfigError(f"mask_ratio out of [0, 1]: {self.mask_ratio}")
        if self.mask_ratio > 0.0 and self.res % self.patch != 0:
            raise ConfigError(f"mask_ratio set but patch {self.patch} does not divide res {self.res}")
        if self.out_dtype not in ("float32", "bfloat16"):
            raise ConfigError(f"out_dtype must be float32 or bfloat16, got {self.out_dtype!r}")
        if self.world_size < 1 or not 0 <= self.rank < self.world_size:
            raise ConfigError(f"bad rank/world_size {self.rank}/{self.world_size}")
        if self.staging not in ("gather", "copy"):
            raise ConfigError(f"staging must be gather or copy, got {self.staging!r}")
        if self.streams < 1 or self.prefetch < 1:
            raise ConfigError("streams and prefetch must be >= 1")
        if self.group < 1:
            raise ConfigError("group must be >= 1")
        if not 0 <= self.fill_chain <= 1024:
            raise ConfigError("fill_chain must be in [0, 1024]")
        if self.visible and self.mask_ratio <= 0.0:
            raise ConfigError("visible tokens need mask_ratio > 0")
        if self.shard_mode not in ("pad", "drop", "stride"):
            raise ConfigError(f"shard_mode must be pad, drop or stride, got {self.shard_mode!r}")


class _HostRing:
    """Pinned host buffers reused round-robin by one stream's batches
    (indices, labels, per-image results), so the hot loop never allocates
    page-locked memory."""

    def __init__(self, depth: int, batch: int, result_words: int):
        import torch
        self.depth = depth
        # indices then labels of a batch of b, contiguous: one H2D copy
        self.il = [torch.empty(2 * batch, dtype=torch.int64, pin_memory=True) for _ in range(depth)]
        self.il_np = [t.numpy() for t in self.il]
        self.res = [torch.empty((batch, result_words), dtype=torch.int32, pin_memory=True)
                    for _ in range(depth)]
        self.ev = [torch.cuda.Event() for _ in range(depth)]
        self.used = [False] * depth
        self.next = 0
        self._views: dict = {}

    def results(self, slot: int, b: int):
        """(pinned tensor, numpy view) of slot's first b result rows."""
        v = self._views.get((slot, b))
        if v is None:
            t = self.res[slot][:b]
            v = self._views[(slot, b)] = (t, t.numpy())
        return v

    def take(self):
        i = self.next
        self.next = (i + 1) % self.depth
        if self.used[i]:
            self.ev[i].synchronize()  # the batch that used this slot is done
        self.used[i] = True
        return i


@dataclass
class _Pending:
    batch: ImageBatch
    samples: np.ndarray | None  # None: descriptors were built natively (rebuilt on error)
    indices: np.ndarray
    results_host: object
    event: object
    epoch: int = 0
    keep: list = field(default_factory=list)
    results_np: object = None  # numpy view of results_host (fast path)
    last: bool = True  # the last batch of its launch set (_enqueue_group)


class Loader:
    """Epoch iterator over a container with the GPU sample pipeline
    (pipeline.py:173-267).  Rank r of a DDP job iterates perm[r::world]."""

    def __init__(self, config: LoaderConfig, container: ContainerHandle | None = None,
                 engine=None):
        import torch
        config.validate()
        self.config = config
        self.handle = container if container is not None else open_container(config.data)
        self._own_handle = container is None
        self.handle.validate_all()
        self.rrc = RrcConfig(tuple(config.scale), tuple(config.ratio), config.res)
        self.aug_level = AugLevel(config.aug)
        self.mask_spec = (MaskSpec.from_resolution(config.res, config.patch, config.mask_ratio)
                          if config.mask_ratio > 0.0 else None)
        from .engine import Engine
        dev = config.device
        if dev is None:
            dev = f"cuda:{torch.cuda.current_device()}"
        w, h = self.handle.max_dims()
        # one libessl context (own scratch) + one CUDA stream per batch in
        # flight: consecutive batches overlap on the GPU
        self._engines = [engine] if engine is not None else []
        while len(self._engines) < config.streams:
            self._engines.append(Engine(dev, max_batch=config.batch_size * config.group,
                                        max_side=max(w, h, 16),
                                        max_payload=self.handle.max_payload()))
        self.engine = self._engines[0]
        self.device = self.engine.device
        self._streams = [torch.cuda.Stream(self.device) for _ in self._engines]
        self._rings = [_HostRing(2 * max(config.prefetch, config.streams) + 2, config.batch_size * config.group,
                                 ctypes.sizeof(N.EsslResult) // 4) for _ in self._engines]
        self._rr = 0
        self.workers = config.workers if config.workers > 0 else (os.cpu_count() or 1)
        rec = self.handle.records
        self._widths = np.ascontiguousarray(rec["width"], np.uint16)
        self._heights = np.ascontiguousarray(rec["height"], np.uint16)
        self._offsets = np.ascontiguousarray(rec["payload_offset"], np.uint64)
        self._lengths = np.ascontiguousarray(rec["payload_length"], np.uint32)
        self._crcs = np.ascontiguousarray(rec["checksum"], np.uint32)
        self._labels_np = rec["label"].astype(np.int64)
        self._blob = self.handle.to_device(self.device) if config.resident else None
        self._pinned_base = (self.handle.pinned_host()
                             if not config.resident and config.staging == "gather" else 0)
        self._host_base = (int(self.handle.bytes.ctypes.data)
                           if not config.resident and config.staging == "copy" else 0)
        self._slots = [0] * len(self._engines)
        self._out_ring: dict = {}
        self._out_next = [0] * len(self._engines)
        self._out_dtype = torch.bfloat16 if config.out_dtype == "bfloat16" else torch.float32
        # the record table, copied once into the native batch planner
        self._ds = ctypes.c_void_p()
        N.check(N.lib().essl_dataset_create(len(self._offsets), N.ptr(self._offsets),
                                            N.ptr(self._lengths), N.ptr(self._crcs),
                                            N.ptr(self._widths), N.ptr(self._heights),
                                            N.ptr(self._labels_np), ctypes.byref(self._ds)),
                "essl_dataset_create")
        self._bcfg = N.EsslBatchCfg()
        self._bio = N.EsslBatchIo()
        # enqueue fast path: byref handles, raw stream handles, per output-slot
        # pointer sets (reuse_outputs), config fields refreshed on retarget
        self._bcfg_ref = ctypes.byref(self._bcfg)
        self._bio_ref = ctypes.byref(self._bio)
        self._st_ptr = [ctypes.c_void_p(s_.cuda_stream) for s_ in self._streams]
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        n_st = len(self._engines)
        self._R = max(2, -(-(max(config.prefetch, n_st) + 2) // n_st))
        self._fast: dict = {}
        self._chain = 0  # essl_batch_io.stage_chain of the next enqueues (the iterators' fill)
        self._refresh_cfg()

    @classmethod
    def from_document(cls, doc) -> "Loader":
        return cls(LoaderConfig.from_document(doc))

    def __len__(self) -> int:
        return len(self.handle)

    def _shard_len(self) -> int:
        c = self.config
        return shard_len(len(self.handle), c.rank, c.world_size, c.shard_mode)

    @property
    def batches_per_epoch(self) -> int:
        return -(-self._shard_len() // self.config.batch_size)

    def retarget(self, res: int | None = None, mask_ratio: float | None = None,
                 scale=None) -> None:
        """Switch progressive-training stage (schedule.py params_for_epoch)
        without reallocating the context or the resident dataset."""
        cfg = self.config
        if res is not None:
            cfg.res = int(res)
        if mask_ratio is not None:
            cfg.mask_ratio = float(mask_ratio)
        if scale is not None:
            cfg.scale = (float(scale[0]), float(scale[1]))
        cfg.validate()
        self.rrc = RrcConfig(tuple(cfg.scale), tuple(cfg.ratio), cfg.res)
        self.mask_spec = (MaskSpec.from_resolution(cfg.res, cfg.patch, cfg.mask_ratio)
                          if cfg.mask_ratio > 0.0 else None)
        self._fast.clear()
        self._refresh_cfg()

    def _refresh_cfg(self) -> None:
        """The batch config fields that only change with the loader config."""
        import torch
        cfg = self.config
        c = self._bcfg
        c.seed = cfg.seed & (2**64 - 1)
        c.scale[0], c.scale[1] = self.rrc.scale
        c.ratio[0], c.ratio[1] = self.rrc.ratio
        c.res = cfg.res
        c.out_kind = N.ESSL_OUT_BF16_NCHW if self._out_dtype == torch.bfloat16 else N.ESSL_OUT_F32_NCHW
        c.check_crc = 1
        T = k = 0
        if self.mask_spec is not None:
            T, k = self.mask_spec.tokens, self.mask_spec.masked_count
        c.tokens, c.masked, c.patch = T, k, cfg.patch
        io = self._bio
        if self._blob is not None:
            io.blob, io.pinned_base, io.stage_slot = self._blob.data_ptr(), None, 0
        else:
            io.blob, io.pinned_base = None, self._pinned_base

    def close(self) -> None:
        if getattr(self, "_ds", None):
            N.lib().essl_dataset_destroy(self._ds)
            self._ds = ctypes.c_void_p()
        if self._own_handle:
            self.handle.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------
    def _descriptors(self, epoch: int, idxs: np.ndarray):
        """Per-sample descriptors: rect + flip (+ 3-Aug draws, blur weights
        filled) from each sample's pipeline stream (pipeline.py:221-227)."""
        from . import augment
        cfg = self.config
        s = self.engine.samples(len(idxs))
        s["offset"] = self._offsets[idxs]
        s["length"] = self._lengths[idxs]
        s["crc32"] = self._crcs[idxs]
        s["check_crc"] = 1
        aug = None
        if self.aug_level is AugLevel.SIMPLE:
            N.check(N.lib().essl_rrc_batch(cfg.seed & (2**64 - 1), epoch & (2**64 - 1),
                                           N.ptr(idxs), len(idxs), N.ptr(self._widths),
                                           N.ptr(self._heights), self.rrc.scale[0],
                                           self.rrc.scale[1], self.rrc.ratio[0],
                                           self.rrc.ratio[1], N.ptr(s)), "essl_rrc_batch")
        else:
            aug = augment.new_aug(len(idxs))
            N.check(N.lib().essl_aug_batch(cfg.seed & (2**64 - 1), epoch & (2**64 - 1),
                                           N.ptr(idxs), len(idxs), N.ptr(self._widths),
                                           N.ptr(self._heights), self.rrc.scale[0],
                                           self.rrc.scale[1], self.rrc.ratio[0],
                                           self.rrc.ratio[1], augment.level_code(self.aug_level),
                                           N.ptr(s), N.ptr(aug)), "essl_aug_batch")
            augment.fill_weights(aug)
        return s, aug

    def _outputs(self, j: int, b: int, pixels=None):
        """This batch's output tensors: caller-provided pixels, the reuse ring
        (R slots per stream, R * streams > the batches in flight beyond the
        one the consumer holds), or fresh tensors."""
        import torch
        cfg = self.config
        n_st = len(self._engines)
        R = max(2, -(-(max(cfg.prefetch, n_st) + 2) // n_st))
        oslot = self._out_next[j] % R
        self._out_next[j] += 1
        dev = self.device
        res = cfg.res

        bmax = cfg.batch_size * cfg.group

        def out(name, shape, dtype):
            if not cfg.reuse_outputs:
                return torch.empty(shape, dtype=dtype, device=dev)
            # one buffer per slot sized for the largest launch set, viewed
            # [:n] (single batches, groups and partial batches share it: no
            # allocation mid-run); keyed by the per-image shape too, so
            # progressive stages (retarget) keep their own rings
            full = (shape[0] // b * bmax,) + tuple(shape[1:])
            key = (j, oslot, name, full, dtype)
            t = self._out_ring.get(key)
            if t is None:
                t = torch.empty(full, dtype=dtype, device=dev)
                self._out_ring[key] = t
            return t[:shape[0]]

        o = {}
        if pixels is not None:
            if tuple(pixels.shape) != (b, 3, res, res) or pixels.dtype != self._out_dtype or \
                    pixels.device != dev or pixels.stride()[1:] != (res * res, res, 1):
                raise ValueError(f"pixels buffer must be {self._out_dtype} [{b},3,{res},{res}] on "
                                 f"{dev} with dense planes")
            o["pixels"] = pixels
        else:
            o["pixels"] = out("pixels", (b, 3, res, res), self._out_dtype)
        o["u8"] = out("u8", (b, res, res, 3), torch.uint8) if cfg.keep_uint8 else None
        o["results"] = out("results", (b, ctypes.sizeof(N.EsslResult) // 4), torch.int32)
        o["il"] = out("il", (2 * b,), torch.int64)
        if self.mask_spec is not None:
            T, k = self.mask_spec.tokens, self.mask_spec.masked_count
            o["mask"] = out("mask", (b, k), torch.int32)
            o["keep"] = out("keep", (b, T - k), torch.int64)
            o["restore"] = out("restore", (b, T), torch.int64)
            if cfg.visible:
                o["tokens"] = out("tokens", (b, T - k, cfg.patch * cfg.patch * 3), torch.bfloat16)
        return o

    def enqueue(self, epoch: int, idxs: np.ndarray, pixels=None) -> _Pending:
        """Issue one batch on the device (asynchronous, on the next of the
        loader's streams): ONE native call (essl_batch_enqueue) builds the
        descriptors (RRC + flip draws), uploads indices/labels, gathers host
        payloads when the container is not resident, runs the mask and the
        decode/resize kernels and downloads the per-image results.
        ``pixels``: optional caller-owned output buffer [b,3,res,res] (e.g. a
        slice of the model's input buffer) written in place of the ring."""
        import torch
        cfg = self.config
        if self._blob is None and cfg.staging == "copy":
            return self._enqueue_py(epoch, idxs, pixels)
        j = self._rr
        self._rr = (j + 1) % len(self._engines)
        eng, st = self._engines[j], self._streams[j]
        idxs = np.ascontiguousarray(idxs, np.int64)
        b = len(idxs)
        o, ptrs, views = self._slot_outputs(j, b, pixels)
        ring = self._rings[j]
        slot = ring.take()  # the batch that last used this slot has completed
        res_host, res_np = ring.results(slot, b)
        aug = None
        if self.aug_level is not AugLevel.SIMPLE:
            _, aug = self._descriptors(epoch, idxs)
        self._bcfg.epoch = epoch & (2**64 - 1)
        io = self._bio
        if self._blob is None:
            io.stage_slot = self._slots[j]
            io.stage_chain = self._chain
            self._slots[j] ^= 1
        io.aug = None if aug is None else aug.ctypes.data
        (io.pixels, io.pixel_stride, io.u8, io.index_label, io.mask, io.ids_keep, io.ids_restore,
         io.tokens, io.results) = ptrs
        io.results_host = res_host.data_ptr()
        # the consumer's stream: its work so far (reads of recycled outputs)
        # completes before this batch's work on st (natively: event + wait)
        io.wait_stream = torch._C._cuda_getCurrentRawStream(self._dev_index)
        rc = N.lib().essl_batch_enqueue(eng._ctx, self._ds, self._bcfg_ref, idxs.ctypes.data, b,
                                        self._bio_ref, self._st_ptr[j])
        if rc:
            N.check(rc, "essl_batch_enqueue")
        if not cfg.reuse_outputs and pixels is None:  # fresh tensors: tell the allocator about st
            for t in o.values():
                if t is not None:
                    t.record_stream(st)
        ev = ring.ev[slot]
        ev.record(st)
        batch = ImageBatch(o["pixels"], views[0], views[1], epoch, o.get("mask"), o["u8"], o.get("keep"),
                           o.get("restore"), o.get("tokens"))
        return _Pending(batch, None, idxs, res_host, ev, epoch, results_np=res_np)

    def _slot_outputs(self, j: int, b: int, pixels=None):
        """This batch's outputs (_outputs), their raw pointers in essl_batch_io
        order and the label / index views -- cached per output-ring slot."""
        cfg = self.config
        key = None
        if cfg.reuse_outputs and pixels is None:
            key = (j, self._out_next[j] % self._R, b)
            hit = self._fast.get(key)
            if hit is not None:
                self._out_next[j] += 1
                return hit
        o = self._outputs(j, b, pixels)

        def dp(name):
            t = o.get(name)
            return None if t is None else t.data_ptr()

        px = o["pixels"]
        ptrs = (px.data_ptr(), int(px.stride()[0]), dp("u8"), o["il"].data_ptr(), dp("mask"), dp("keep"),
                dp("restore"), dp("tokens"), o["results"].data_ptr())
        il = o["il"]
        rec = (o, ptrs, (il[b:], il[:b]))
        if key is not None:
            self._fast[key] = rec
        return rec

    def _enqueue_py(self, epoch: int, idxs: np.ndarray, pixels=None) -> _Pending:
        """Host-thread staging path (staging="copy"): descriptors in numpy,
        payloads gathered by host threads into a pinned ring, then the
        decode / mask calls one by one."""
        import torch
        cfg = self.config
        j = self._rr
        self._rr = (j + 1) % len(self._engines)
        eng, st = self._engines[j], self._streams[j]
        st.wait_stream(torch.cuda.current_stream(self.device))
        idxs = np.ascontiguousarray(idxs, np.int64)
        b, res = len(idxs), cfg.res
        samples, aug = self._descriptors(epoch, idxs)
        ptrs = samples["offset"] + np.uint64(self._host_base)
        blob_ptr = eng.stage(self._slots[j], ptrs, samples["length"].copy(), samples,
                             nthreads=min(8, self.workers), stream=st)
        self._slots[j] ^= 1
        ring = self._rings[j]
        slot = ring.take()
        o = self._outputs(j, b, pixels)
        kind = N.ESSL_OUT_BF16_NCHW if self._out_dtype == torch.bfloat16 else N.ESSL_OUT_F32_NCHW
        hil, hil_np, res_host = ring.il[slot], ring.il_np[slot], ring.res[slot][:b]
        hil_np[:b] = idxs
        hil_np[b:2 * b] = self._labels_np[idxs]
        il = o["il"]
        sp = ctypes.c_void_p(st.cuda_stream)
        L = N.lib()
        N.check(L.essl_memcpy_async(N.ptr(il), N.ptr(hil), 16 * b, sp), "essl_memcpy_async")
        indices, labels = il[:b], il[b:]
        if self.mask_spec is not None:
            T, k = self.mask_spec.tokens, self.mask_spec.masked_count
            eng.mask(cfg.seed, epoch, indices, T, k, o["mask"], o["keep"], o["restore"], stream=st)
        eng.decode_rrc(blob_ptr, samples, res, kind, o["pixels"], o["u8"], o["results"], stream=st,
                       aug=aug, out_stride=int(o["pixels"].stride()[0]),
                       vis=(cfg.patch, o.get("restore"), o.get("tokens")))
        N.check(L.essl_memcpy_async(N.ptr(res_host), N.ptr(o["results"]), o["results"].numel() * 4, sp),
                "essl_memcpy_async")
        if not cfg.reuse_outputs and pixels is None:
            for t in o.values():
                if t is not None:
                    t.record_stream(st)
        ev = ring.ev[slot]
        ev.record(st)
        batch = ImageBatch(o["pixels"], labels, indices, epoch, o.get("mask"), o["u8"], o.get("keep"),
                           o.get("restore"), o.get("tokens"))
        return _Pending(batch, samples, idxs, res_host, ev, epoch)

    def join(self, p: _Pending) -> None:
        """Make the consumer stream wait for a batch (no host sync)."""
        import torch
        torch.cuda.current_stream(self.device).wait_event(p.event)

    def finish(self, p: _Pending) -> ImageBatch:
        """Wait for a batch and raise the reference exception on failure."""
        self.join(p)
        p.event.synchronize()
        r = p.results_np if p.results_np is not None else p.results_host.numpy()
        if r[:, 0].any():
            samples = p.samples if p.samples is not None else self._descriptors(p.epoch, p.indices)[0]
            self.engine.raise_for(r, samples, p.indices)
        return p.batch

    @property
    def engines(self):
        return list(self._engines)

    def set_option(self, option: int, value: int) -> None:
        """libessl context option (include/essl.h ESSL_OPT_*) on every stream."""
        for e in self._engines:
            e.set_option(option, value)

    @property
    def launches(self) -> int:
        return sum(e.launches for e in self._engines)

    def profile_read(self) -> dict:
        tot: dict = {}
        for e in self._engines:
            for k, (ms, n) in e.profile_read().items():
                a, b = tot.get(k, (0.0, 0))
                tot[k] = (a + ms, b + n)
        return tot

    def _plan(self, epoch: int):
        cfg = self.config
        perm = shard(epoch_permutation(cfg.seed, epoch, len(self.handle)), cfg.rank,
                     cfg.world_size, cfg.shard_mode)
        B = cfg.batch_size
        for s in range(0, len(perm), B):
            yield epoch, perm[s:s + B]

    def _run(self, plan, into=None):
        """Keep `depth` launch sets in flight over the (epoch, indices) plan
        (one batch each, or up to `group` batches of one epoch each)."""
        q: deque = deque()
        depth = max(self.config.prefetch, len(self._engines))
        if into is not None and len(into) < depth + 1:
            raise ValueError(f"into: need at least {depth + 1} buffers for {depth} batches in flight")
        G = self.config.group if into is None else 1
        it = iter(plan)
        held = []  # a plan item read ahead that starts the next group
        nb = 0

        def take(g):
            """The next launch set: [(epoch, indices), ...] (empty at the end)."""
            items = [held.pop()] if held else []
            while len(items) < g:
                nxt = next(it, None)
                if nxt is None:
                    break
                if items and nxt[0] != items[0][0]:  # groups stay within an epoch
                    held.append(nxt)
                    break
                items.append(nxt)
            return items

        def issue(items):
            nonlocal nb
            if len(items) > 1:
                return self.enqueue_group(items[0][0], [i for _, i in items])
            e, idxs = items[0]
            buf = None
            if into is not None:
                buf = into[nb % len(into)]
                buf = buf[:len(idxs)] if buf.shape[0] != len(idxs) else buf
            nb += 1
            return [self.enqueue(e, idxs, buf)]

        # the pipeline fills with single batches (the first results come back
        # soonest); groups take over once `depth` sets are in flight
        sets = 0
        # host-staged payloads: the fill's bus gathers run oldest first
        self._chain = self.config.fill_chain if self._blob is None else 0
        try:
            while sets < depth:
                items = take(1)
                if not items:
                    break
                q.extend(issue(items))
                sets += 1
        finally:
            self._chain = 0
        while q:
            p = q.popleft()
            if p.last:  # its launch set is done with: issue the next one
                items = take(G)
                if items:
                    q.extend(issue(items))
            yield self.finish(p)

    def enqueue_group(self, epoch: int, parts: list) -> list:
        """Consecutive batches of one epoch in ONE launch set (one native
        call over their concatenated indices; at most `group` of them); each
        batch's outputs are views of the set's ring buffers.  Returns one
        pending batch per part, in order (finish / join each)."""
        if sum(len(p) for p in parts) > self.config.batch_size * self.config.group:
            raise ValueError("enqueue_group: more images than batch_size * group")
        idxs = np.concatenate([np.asarray(p, np.int64) for p in parts])
        p = self.enqueue(epoch, idxs)
        g = p.batch
        out, off = [], 0
        for k, part in enumerate(parts):
            b = len(part)
            sl = slice(off, off + b)

            def v(t):
                return None if t is None else t[sl]
            batch = ImageBatch(g.pixels[sl], g.labels[sl], g.indices[sl], epoch, v(g.mask), v(g.uint8),
                               v(g.ids_keep), v(g.ids_restore), v(g.visible))
            out.append(_Pending(batch, None, idxs[sl], p.results_host[sl], p.event, epoch,
                                results_np=p.results_np[sl] if p.results_np is not None else None,
                                last=k == len(parts) - 1))
            off += b
        return out

    def epoch(self, epoch: int, into=None):
        """Yield the batches of one epoch (this rank's shard) in permutation order.

        ``into``: optional sequence of caller-owned pixel buffers
        [batch_size,3,res,res] (e.g. the model's input buffers), used round
        robin; a batch's pixels are written straight into its buffer, which
        must not be reused before the batch has been consumed (pass at least
        prefetch + 2 buffers)."""
        return self._run(self._plan(epoch), into)

    def epochs(self, first: int, count: int | None = None, into=None, steps: int | None = None):
        """Batches of epochs first, first+1, ... (count of them, or without
        end) with the prefetch pipeline kept full across epoch boundaries --
        the same batches as consecutive epoch() calls, without the drain /
        refill bubble at each boundary (a persistent-worker DataLoader).
        ``steps``: stop after that many batches (nothing is decoded ahead
        past the last one -- a training run of a fixed step count)."""
        import itertools
        es = itertools.count(first) if count is None else range(first, first + count)
        plan = itertools.chain.from_iterable(self._plan(e) for e in es)
        if steps is not None:
            plan = itertools.islice(plan, steps)
        return self._run(plan, into)
